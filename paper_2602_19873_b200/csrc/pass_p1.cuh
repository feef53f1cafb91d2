// Mixed-precision pass for point clusters (ClusterParams(1, 1, w), gather), SURVEY
// §8(f4); included by pass.cu after pass_item.cuh. An SC is 64 one-particle i-clusters;
// an entry is one j particle with a 64-bit mask over the i.
//
// Warp per SC (dynamic counter); lane = (i, i + 32): each lane owns two i particles and
// walks the entries in order (ascending j, the reference's order), so the i sums stay in
// registers. Per 32 entries the j particles are staged relative to the SC's first
// particle in hi + lo fp32 (coordinate error ~2^-48: the guard band is the fp32
// arithmetic's); the lane's two slots run as one f32x2 pair. Cutoff against the per-i
// guard band [lo, hi]; band slots take the reference's fp64 predicate and kernel, LJ
// pairs closer than kLjClose fp64 from the staged hi/lo; the density spline is
// evaluated in fp64 from the hi/lo difference (a point-cluster list has few slots, and
// the spline's support edge amplifies distance errors by 3 / (1 - q)).
struct alignas(16) P1pSmem {
    float jx[32], jy[32], jz[32], jlx[32], jly[32], jlz[32];
    unsigned long long jmask[32];
    uint32_t idx[64];
};

template <int K>
__global__ void __launch_bounds__(kPiWarps * 32, 4) k_pass_p1(const __grid_constant__ PassArgs A,
                                                             unsigned long long* __restrict__ work) {
    constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    constexpr int NO = nout<K>();
    extern __shared__ __align__(16) unsigned char dsm[];
    P1pSmem& S = reinterpret_cast<P1pSmem*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    const uint32_t w = uint32_t(A.w);
    const float sig2 = float(A.sigma * A.sigma);
    const float close2 = A.lj_close2 * sig2;
    const double sig2d = A.sigma * A.sigma, eps24d = 24.0 * A.eps, eps4d = 4.0 * A.eps;

    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        const uint64_t sc = A.sc_begin + __shfl_sync(0xffffffffu, t, 0);
        if (sc >= A.num_sc) break;
        const uint32_t count = A.counts[sc];
        const uint8_t* rec = nullptr;
        const uint8_t* idata = nullptr;
        uint64_t ilen = 0;
        bool bad = false;
        if (count) {
            const uint64_t begin = A.offsets[sc], end = A.offsets[sc + 1];
            const uint64_t mb = uint64_t(count) * 8;
            if (begin + mb > end) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgMaskSlice, begin);
                bad = true;
            } else {
                rec = A.blob + begin;
                idata = rec + mb;
                ilen = end - begin - mb;
                if (!A.compress && ilen != uint64_t(count) * 4) {
                    if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgRawLen, ilen);
                    bad = true;
                }
            }
        }
        // ---- the lane's two i (hi + lo relative to the SC's first particle)
        const uint64_t p0 = sc * kSC;
        const uint32_t np = uint32_t(tmin<uint64_t>(p0 + kSC, A.n) - p0);
        const double ox = A.x[p0], oy = A.y[p0], oz = A.z[p0];
        auto rel = [&](double v, double o, int d) {
            double r = dsub(v, o);
            if (A.box.per[d]) {
                const double L = A.box.len[d];
                if (r > 0.5 * L) r = dsub(r, L);
                else if (r < -0.5 * L) r = dadd(r, L);
            }
            return r;
        };
        float hx[2], hy[2], hz[2], lx[2], ly[2], lz[2], tlo[2], thi[2];
        double hh[2], isc[2];
        float eax = 0.f, eay = 0.f, eaz = 0.f, er = 0.f;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const uint32_t k = lane + 32u * s;
            hx[s] = hy[s] = hz[s] = lx[s] = ly[s] = lz[s] = 0.f, tlo[s] = thi[s] = -1.f, hh[s] = 1.0;
            if (k < np) {
                const double qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                hx[s] = float(qx), hy[s] = float(qy), hz[s] = float(qz);
                lx[s] = float(qx - double(hx[s])), ly[s] = float(qy - double(hy[s])), lz[s] = float(qz - double(hz[s]));
                hh[s] = A.h[p0 + k];
                const double r = dmul(A.qs, hh[s]), r2 = dmul(r, r);
                eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                er = fmaxf(er, float(r));
                // hi + lo coordinates: the difference error is the fp32 arithmetic's (2^-24 r term)
                const double ex = 5.9604644775390625e-08 * r;
                const double g = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
                tlo[s] = __double2float_rd(r2 - g), thi[s] = __double2float_ru(r2 + g);
            }
            isc[s] = 8.0 / (kPi * hh[s] * hh[s] * hh[s]);
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
        const bool unsafe = (A.box.per[0] && double(eax) + double(er) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(er) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(er) >= 0.49 * A.box.len[2]);
        const f2 xi2 = f2p(hx[0], hx[1]), yi2 = f2p(hy[0], hy[1]), zi2 = f2p(hz[0], hz[1]);
        const f2 lxi2 = f2p(lx[0], lx[1]), lyi2 = f2p(ly[0], ly[1]), lzi2 = f2p(lz[0], lz[1]);
        double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        uint32_t cnt[2] = {0, 0};
        bool coincident = false;
        uint64_t pos = 0, running = 0;
        for (uint32_t bb = 0; !bad && bb < count; bb += w) {
            const uint32_t len = tmin<uint32_t>(w, count - bb);
            if (A.compress) {
                uint64_t off = 0;
                int msg = 0;
                const uint64_t np2 = warp_decode_block(idata, ilen, pos, len, int(w), running, S.idx, &off, &msg);
                if (np2 == ~0ull) {
                    if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off);
                    bad = true;
                    break;
                }
                pos = np2;
                if (bb + len == count && pos != ilen) {
                    if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, pos);
                    bad = true;
                    break;
                }
            } else {
                for (uint32_t k = lane; k < len; k += 32) {
                    const uint8_t* p = idata + 4ull * (bb + k);
                    S.idx[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
                }
            }
            if (A.g2l)  // domain decomposition: stored global ids -> local clusters (same lanes as the decode)
                for (uint32_t k = lane; k < len; k += 32) S.idx[k] = A.g2l[S.idx[k]];
            __syncwarp();
            for (uint32_t h0 = 0; h0 < len; h0 += 32) {
                const uint32_t n = tmin<uint32_t>(32, len - h0);
                if (lane < n) {  // stage entry `lane` (hi + lo) and its mask
                    const uint64_t j = S.idx[h0 + lane];
                    const uint8_t* r8 = rec + 8ull * (bb + h0 + lane);
                    unsigned long long m = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) m |= (unsigned long long)r8[q] << (8 * q);
                    float fx = kFar, fy = kFar, fz = kFar, gx = 0.f, gy = 0.f, gz = 0.f;
                    if (j < A.n) {
                        const double qx = rel(A.x[j], ox, 0), qy = rel(A.y[j], oy, 1), qz = rel(A.z[j], oz, 2);
                        fx = float(qx), fy = float(qy), fz = float(qz);
                        gx = float(qx - double(fx)), gy = float(qy - double(fy)), gz = float(qz - double(fz));
                    } else {
                        m = 0;
                    }
                    S.jx[lane] = fx, S.jy[lane] = fy, S.jz[lane] = fz, S.jlx[lane] = gx, S.jly[lane] = gy, S.jlz[lane] = gz;
                    S.jmask[lane] = m;
                }
                __syncwarp();
                float fa[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};  // the chunk's fp32 sums per slot
                for (uint32_t e = 0; e < n; ++e) {
                    const unsigned long long m = S.jmask[e];
                    const bool b0 = (m >> lane) & 1ull, b1 = (m >> (lane + 32)) & 1ull;
                    if (!__any_sync(0xffffffffu, b0 | b1)) continue;
                    const uint64_t gj = S.idx[h0 + e];
                    const float jxh = S.jx[e], jyh = S.jy[e], jzh = S.jz[e];
                    const f2 dx = f2add(f2sub(xi2, f2p(jxh, jxh)), f2sub(lxi2, f2p(S.jlx[e], S.jlx[e])));
                    const f2 dy = f2add(f2sub(yi2, f2p(jyh, jyh)), f2sub(lyi2, f2p(S.jly[e], S.jly[e])));
                    const f2 dz = f2add(f2sub(zi2, f2p(jzh, jzh)), f2sub(lzi2, f2p(S.jlz[e], S.jlz[e])));
                    float d2[2];
                    f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2[0], d2[1]);
                    float dxs[2], dys[2], dzs[2];
                    f2u(dx, dxs[0], dxs[1]);
                    f2u(dy, dys[0], dys[1]);
                    f2u(dz, dzs[0], dzs[1]);
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        if (!(s ? b1 : b0)) continue;
                        const uint64_t gi = p0 + lane + 32u * s;
                        if (gi == gj) continue;
                        const bool in = d2[s] < tlo[s];
                        const bool special = unsafe || (!in && d2[s] <= thi[s]) || (LJ && in && d2[s] < close2);
                        if (!special) {
                            if (!in) continue;
                            ++cnt[s];
                            if (K == SFCNL_KERNEL_DENSITY) {
                                // fp64 spline from the hi + lo difference
                                const double ddx = (double(hx[s]) - double(jxh)) + (double(lx[s]) - double(S.jlx[e]));
                                const double ddy = (double(hy[s]) - double(jyh)) + (double(ly[s]) - double(S.jly[e]));
                                const double ddz = (double(hz[s]) - double(jzh)) + (double(lz[s]) - double(S.jlz[e]));
                                const double q = sqrt(ddx * ddx + ddy * ddy + ddz * ddz) / hh[s];
                                const double tt = fmax(1.0 - q, 0.0), uu = fmax(0.5 - q, 0.0);
                                acc[s][0] += A.m[gj] * (2.0 * isc[s]) * (tt * tt * tt - 4.0 * uu * uu * uu);
                            } else if (LJ) {
                                const float inv2 = 1.f / d2[s], s2 = sig2 * inv2, s6 = s2 * s2 * s2;
                                float coef = inv2 * s6 * (2.f * s6 - 1.f), en = s6 * (s6 - 1.f);
                                if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                    coef *= float(eps24d), en *= float(eps4d);
                                    const float qq = float(A.ck * A.q[gi] * A.q[gj]), ir = rsqrtf(d2[s]);
                                    en += qq * ir;
                                    coef += qq * ir * inv2;
                                }
                                fa[s][0] += coef * dxs[s], fa[s][1] += coef * dys[s], fa[s][2] += coef * dzs[s], fa[s][3] += en;
                            }
                            continue;
                        }
                        // special: close LJ pair (fp64 from hi + lo) or the reference predicate + fp64 kernel
                        double v[4];
                        bool done = false;
                        if (LJ && !unsafe && in) {
                            const double ddx = (double(hx[s]) - double(jxh)) + (double(lx[s]) - double(S.jlx[e]));
                            const double ddy = (double(hy[s]) - double(jyh)) + (double(ly[s]) - double(S.jly[e]));
                            const double ddz = (double(hz[s]) - double(jzh)) + (double(lz[s]) - double(S.jlz[e]));
                            const double dd2 = ddx * ddx + ddy * ddy + ddz * ddz;
                            if (dd2 >= double(kLjTiny2) * sig2d) {
                                const double inv2 = 1.0 / dd2, s2 = sig2d * inv2, s6 = s2 * s2 * s2;
                                double coef = eps24d * inv2 * s6 * (2.0 * s6 - 1.0);
                                double en = eps4d * s6 * (s6 - 1.0);
                                if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                    const double qq = A.ck * A.q[gi] * A.q[gj], ir = sqrt(inv2);
                                    en += qq * ir;
                                    coef += qq * ir * inv2;
                                }
                                v[0] = coef * ddx, v[1] = coef * ddy, v[2] = coef * ddz, v[3] = en;
                                done = true;
                            }
                        }
                        if (!done) {
                            const double hi_ = hh[s], r = dmul(A.qs, hi_);
                            double ex, ey, ez;
                            const double dd2 = pair_d2_exact(A.x[gi], A.y[gi], A.z[gi], A.x[gj], A.y[gj], A.z[gj], A.box,
                                                             &ex, &ey, &ez);
                            if (dd2 > dmul(r, r)) continue;
                            if (eval_exact<K>(A, gi, gj, dd2, ex, ey, ez, hi_, v)) {
                                coincident = true;
                                continue;
                            }
                        }
                        ++cnt[s];
#pragma unroll
                        for (int o = 0; o < NO; ++o) acc[s][o] += v[o];
                    }
                }
                if (LJ) {  // the chunk's fp32 sums into the fp64 totals (eps factors for K == LJ)
#pragma unroll
                    for (int s = 0; s < 2; ++s)
#pragma unroll
                        for (int o = 0; o < 4; ++o)
                            acc[s][o] += double(fa[s][o]) * (K == SFCNL_KERNEL_LJ ? (o < 3 ? eps24d : eps4d) : 1.0);
                }
                __syncwarp();
            }
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        if (!bad) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const uint32_t k = lane + 32u * s;
                if (k < np) {
#pragma unroll
                    for (int o = 0; o < NO; ++o) A.out[o][p0 + k] = (K == SFCNL_KERNEL_COUNT) ? double(cnt[s]) : acc[s][o];
                    A.cnt[p0 + k] = cnt[s];
                }
            }
        }
        __syncwarp();
    }
}
