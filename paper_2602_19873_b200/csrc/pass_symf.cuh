// Symmetric (half-list) mixed-precision pass (precision 1, ci == 8, cj in {4, 8}),
// every stored pair is evaluated ONCE and feeds both particles, which
// is the point of the half list (paper §II-D; reduce.hpp:186-194 i side + j-side
// accumulators). Included by pass.cu after pass_warp.cuh / pass_sym.cuh.
//
// Warp per super-cluster (dynamic counter), staged like k_pass_warp (SC-relative fp32,
// hi + lo for LJ). The loop order is entries outer, i-clusters inner: lane = (i of
// cluster b, j quarter q), two slots per lane (j = q, q + 4).
//  * i side: per (entry, b) the lane's two slots are reduced over the four j-quarter
//    lanes (two xor shuffles) and added into the per-i fp64 sums in shared memory;
//  * j side: the lane keeps its slots' signed sums in registers over all bits b of
//    the entry (reference order: odd outputs negated), reduced over the eight i lanes
//    once per entry and written to jacc[entry][j] (fp32, eps factors applied);
//  * k_sym_fgather then adds, per particle, the jacc of every entry whose j-cluster
//    holds it (the transposed entry lists of pass_sym.cuh), in entry order.
// Cutoff decisions: r_ij = qs max(h_i, h_j); the fp32 test uses max(lo_i, lo_j) and
// max(hi_i, hi_j) (the guard band is monotone in r); band slots and LJ pairs closer
// than kLjClose take fp64 (reference predicate; close pairs from the staged hi/lo).
// Within an entry whose j-cluster overlaps the SC's own particles only j > i is
// evaluated (i == j never; mirror_stored, reduce.hpp:16-21, holds for every i > j
// there). Unsafe SCs evaluate every slot through the reference fp64 predicate.

constexpr int kPsChunk = 16;  // entries staged at a time (smaller than k_pass_warp's: more per-warp state)

template <int K>
struct alignas(16) PsSmem {
    static constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    static constexpr int NO = nout<K>();
    // density: one more channel, the slot's weight in the error bound of the fp32 spline
    static constexpr int NE = NO + (K == SFCNL_KERNEL_DENSITY ? 1 : 0);
    // hi + lo staging for LJ and density (the density spline's edge amplifies distance
    // errors by 3 / (1 - q); the few-neighbour side of a half list cannot average them)
    static constexpr bool HL = LJ || K == SFCNL_KERNEL_DENSITY;
    float sj[kPsChunk * 4 * (HL ? 12 : 8)];  // as PwSmem (LJ layout when HL)
    float2 sm[K == SFCNL_KERNEL_DENSITY ? kPsChunk * 4 : 1];  // density: m of slots {a, b}
    float2 jlo[kPsChunk * 4], jhi[kPsChunk * 4];  // per (entry, quarter): thresholds of slots {a, b}
    uint32_t idx[64];
    float ix[64], iy[64], iz[64];
    float ilx[HL ? 64 : 1], ily[HL ? 64 : 1], ilz[HL ? 64 : 1];
    float iscale[64];  // density: 8 / (pi h^3)
    float iinvh[64];
    double acc[64][NE];
    uint32_t cnt[64];
    float ilo[64], ihi[64];
    float jside[kPsChunk][8][NE];  // the chunk's j-side sums (folded scale) per (entry, j)
    uint32_t jsc[kPsChunk][8];
    float ip[64][4][NE];  // the chunk's i-side partial sums per (i, j-quarter lane): lane-private
    float ipc[64][4];
};

constexpr uint32_t kSqCap = kPsChunk * 8 * 64;  // deferred special slots per warp and chunk (worst case)

template <int K>
constexpr size_t ps_smem() {
    return size_t(kPwWarps) * sizeof(PsSmem<K>);
}

// fp64 pair value through the reference predicate (symmetric radius); returns 1 and
// fills v when in range, 0 when not, -1 on coincidence.
template <int K>
__device__ __noinline__ int sym_exact_slot(const PassArgs& A, uint64_t i, uint64_t j, double v[4]) {
    const double hi = A.h[i];
    double dx, dy, dz;
    const double d2 = pair_d2_exact(A.x[i], A.y[i], A.z[i], A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
    const double rr = dmul(A.qs, smax(hi, A.h[j]));
    if (d2 > dmul(rr, rr)) return 0;
    return eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v) ? -1 : 1;
}

template <int K>
constexpr int ps_min_blocks() {
#ifdef SFCNL_SYMW_MINB
    return SFCNL_SYMW_MINB;
#else
    return (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB) ? 3 : 4;  // LJ: 168 registers, no spills
#endif
}

template <int K, int CJ>
__global__ void __launch_bounds__(kPwWarps * 32, ps_min_blocks<K>()) k_pass_symw(const __grid_constant__ PassArgs A,
                                                                unsigned long long* __restrict__ work,
                                                                const uint64_t* __restrict__ ebase, float* __restrict__ jacc,
                                                                uint32_t* __restrict__ jcnt, uint32_t* __restrict__ ejcl,
                                                                uint32_t* __restrict__ squeue, double* __restrict__ aux,
                                                                double* __restrict__ jspec) {
    constexpr bool LJ = PsSmem<K>::LJ;
    constexpr bool HL = PsSmem<K>::HL;
    constexpr int NO = nout<K>();
    constexpr int NE = PsSmem<K>::NE;
    extern __shared__ __align__(16) unsigned char dsm[];
    PsSmem<K>& S = reinterpret_cast<PsSmem<K>*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    const uint32_t il = lane >> 2, jq = lane & 3;
    const uint32_t w = uint32_t(A.w);
    const float sig2 = float(A.sigma * A.sigma);
    const float close2 = A.lj_close2 * sig2;
    uint32_t* const sq = squeue + (uint64_t(blockIdx.x) * kPwWarps + (threadIdx.x >> 5)) * kSqCap;
    const unsigned lt_mask = (1u << lane) - 1u;
    const double sig2d = A.sigma * A.sigma, eps24d = 24.0 * A.eps, eps4d = 4.0 * A.eps;
    // LJ outputs are accumulated without the 24 eps / 4 eps factors (applied at the flushes)
    const float fscale[4] = {K == SFCNL_KERNEL_LJ ? float(eps24d) : 1.f, K == SFCNL_KERNEL_LJ ? float(eps24d) : 1.f,
                             K == SFCNL_KERNEL_LJ ? float(eps24d) : 1.f, K == SFCNL_KERNEL_LJ ? float(eps4d) : 1.f};

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
            const uint64_t mb = uint64_t(count) * A.mask_bytes;
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

        // ---- i side (as k_pass_warp)
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
        float eax = 0.f, eay = 0.f, eaz = 0.f, er = 0.f;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const uint32_t k = lane + 32u * s;
            float fx = 0.f, fy = 0.f, fz = 0.f;
            double r = -1.0, hk = 1.0, qx = 0, qy = 0, qz = 0;
            if (k < np) {
                qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                hk = A.h[p0 + k];
                fx = float(qx), fy = float(qy), fz = float(qz);
                r = dmul(A.qs, hk);
                eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                er = fmaxf(er, float(r));
            }
            S.ix[k] = fx, S.iy[k] = fy, S.iz[k] = fz;
            if (HL) S.ilx[k] = float(qx - double(fx)), S.ily[k] = float(qy - double(fy)), S.ilz[k] = float(qz - double(fz));
            if (K == SFCNL_KERNEL_DENSITY) S.iscale[k] = float(8.0 / (kPi * hk * hk * hk)), S.iinvh[k] = float(1.0 / hk);
#pragma unroll
            for (int o = 0; o < NE; ++o) {
                S.acc[k][o] = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) S.ip[k][q][o] = 0.f;
            }
            S.cnt[k] = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) S.ipc[k][q] = 0.f;
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz);
        // the j side's radius can exceed the i side's: use the global max h for the image test
        const float erj = fmaxf(warp_fmax(er), float(A.qs * A.maxh));
        const bool unsafe = (A.box.per[0] && double(eax) + double(erj) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(erj) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(erj) >= 0.49 * A.box.len[2]);
        const float Ei = fmaxf(eax, fmaxf(eay, eaz));
        __syncwarp();

        bool coincident = false;
        float E_run = -1.f;
        uint64_t pos = 0, running = 0;
        uint32_t qn = 0;  // deferred special slots of the current chunk (warp-uniform)
        const uint64_t gE0 = count ? ebase[sc] : 0;
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
            __syncwarp();
            for (uint32_t h0 = 0; h0 < len; h0 += kPsChunk) {
                const uint32_t n = tmin<uint32_t>(kPsChunk, len - h0);
                const bool have = lane < n;
                const uint32_t my_idx = have ? S.idx[h0 + lane] : 0u;
                const uint32_t my_msk = have ? uint32_t(rec[bb + h0 + lane]) : 0u;
                // ---- stage the chunk's j particles
                float emax = 0.f;
                if (!unsafe) {
#pragma unroll
                    for (int k0 = 0; k0 < kPsChunk / 4; k0 += 4) {
                        double vx[4], vy[4], vz[4], vm[4];
                        bool val[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t e = uint32_t(k0 + u) * 4 + (lane >> 3), jj = lane & 7;
                            const uint32_t ie = __shfl_sync(0xffffffffu, my_idx, e);
                            const uint64_t j = uint64_t(ie) * CJ + jj;
                            val[u] = e < n && jj < uint32_t(CJ) && j < A.n;
                            vx[u] = vy[u] = vz[u] = vm[u] = 0.0;
                            if (val[u]) {
                                vx[u] = A.x[j], vy[u] = A.y[j], vz[u] = A.z[j];
                                if (K == SFCNL_KERNEL_DENSITY) vm[u] = A.m[j];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t e = uint32_t(k0 + u) * 4 + (lane >> 3), jj = lane & 7;
                            if (e >= n) continue;
                            float fx = kFar, fy = kFar, fz = kFar, fm = 0.f, lx = 0.f, ly = 0.f, lz = 0.f;
                            if (val[u]) {
                                const double qx = rel(vx[u], ox, 0), qy = rel(vy[u], oy, 1), qz = rel(vz[u], oz, 2);
                                fx = float(qx), fy = float(qy), fz = float(qz);
                                fm = float(vm[u]);
                                if (HL) lx = float(qx - double(fx)), ly = float(qy - double(fy)), lz = float(qz - double(fz));
                                emax = fmaxf(emax, fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))));
                            }
                            const uint32_t q = jj & 3, hb = (jj < 4 || CJ == 8) ? (jj >> 2) : 1u;
                            if (!(jj < 4 || CJ == 8)) fx = fy = fz = kFar, fm = 0.f, lx = ly = lz = 0.f;
                            if (HL) {
                                float* p = S.sj + (e * 4 + q) * 12 + hb;
                                p[0] = fx, p[2] = fy, p[4] = fz, p[6] = lx, p[8] = ly, p[10] = lz;
                                if constexpr (K == SFCNL_KERNEL_DENSITY) reinterpret_cast<float*>(&S.sm[e * 4 + q])[hb] = fm;
                            } else {
                                float* p = S.sj + (e * 4 + q) * 8 + hb;
                                p[0] = fx, p[2] = fy, p[4] = fz, p[6] = fm;
                            }
                        }
                    }
                }
                const float E = fmaxf(Ei, warp_fmax(emax));
                if (!unsafe && E > E_run) {  // per-i thresholds (guard band of pass.cu)
                    E_run = fmaxf(E, E_run * 1.0625f);
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const uint32_t k = lane + 32u * s;
                        float lo = -1.f, hi = -1.f;
                        if (k < np) {
                            const double r = dmul(A.qs, A.h[p0 + k]), r2 = dmul(r, r);
                            const double ex = 1.1920928955078125e-07 * double(E_run) + 5.9604644775390625e-08 * r;
                            const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
                            lo = __double2float_rd(r2 - guard);
                            hi = __double2float_ru(r2 + guard);
                        }
                        S.ilo[k] = lo, S.ihi[k] = hi;
                    }
                }
                if (!unsafe) {  // per-j thresholds with the same bound (monotone in r: max with the i side's)
#pragma unroll
                    for (int u = 0; u < kPsChunk / 4; ++u) {
                        const uint32_t e = uint32_t(u) * 4 + (lane >> 3), jj = lane & 7;
                        const uint32_t ie = __shfl_sync(0xffffffffu, my_idx, e);
                        const uint64_t j = uint64_t(ie) * CJ + jj;
                        float lo = -1.f, hi = -1.f;
                        if (e < n && jj < uint32_t(CJ) && j < A.n) {
                            const double r = dmul(A.qs, A.h[j]), r2 = dmul(r, r);
                            const double ex = 1.1920928955078125e-07 * double(E_run) + 5.9604644775390625e-08 * r;
                            const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
                            lo = __double2float_rd(r2 - guard);
                            hi = __double2float_ru(r2 + guard);
                        }
                        if (e < n && (jj < 4 || CJ == 8)) {
                            const uint32_t q = jj & 3, hb = jj >> 2;
                            reinterpret_cast<float*>(&S.jlo[e * 4 + q])[hb] = lo;
                            reinterpret_cast<float*>(&S.jhi[e * 4 + q])[hb] = hi;
                        } else if (e < n && jj >= 4 && CJ == 4) {  // dummy slot b
                            reinterpret_cast<float*>(&S.jlo[e * 4 + (jj & 3)])[1] = -1.f;
                            reinterpret_cast<float*>(&S.jhi[e * 4 + (jj & 3)])[1] = -1.f;
                        }
                    }
                }
                __syncwarp();

                for (uint32_t e = 0; e < n; ++e) {
                    const uint32_t m = __shfl_sync(0xffffffffu, my_msk, e);
                    const uint64_t jb = uint64_t(__shfl_sync(0xffffffffu, my_idx, e)) * CJ;
                    const uint64_t ja_g = jb + jq, jb_g = jb + jq + 4;  // the lane's two j (global)
                    if (lane == 0) ejcl[gE0 + bb + h0 + e] = uint32_t(jb / CJ);
                    const bool selfe = jb < p0 + kSC && jb + CJ > p0;   // j-cluster overlaps the SC
                    f2 jv[4] = {0, 0, 0, 0};
                    float jc0 = 0.f, jc1 = 0.f;
                    if (unsafe) {
                        for (uint32_t bits = m; bits; bits &= bits - 1) {
                            const uint32_t b = __ffs(bits) - 1;
                            const uint32_t li = b * 8 + il;
                            const uint64_t i = p0 + li;
                            double vi[4] = {0, 0, 0, 0};
                            uint32_t ci = 0;
                            float ja[4] = {0, 0, 0, 0}, jbv[4] = {0, 0, 0, 0};
                            if (li < np) {
#pragma unroll
                                for (int sl = 0; sl < 2; ++sl) {
                                    const uint64_t j = sl ? jb_g : ja_g;
                                    if ((sl && CJ == 4) || j >= A.n || j <= i) continue;
                                    double v[4];
                                    const int rc = sym_exact_slot<K>(A, i, j, v);
                                    if (rc < 0) coincident = true;
                                    if (rc <= 0) continue;
                                    ++ci;
#pragma unroll
                                    for (int o = 0; o < NO; ++o) {
                                        vi[o] += v[o];
                                        const float sv = float((NO == 4 && o < 3) ? -v[o] : v[o]);
                                        if (sl) jbv[o] += sv;
                                        else ja[o] += sv;
                                    }
                                    if (sl) jc1 += 1.f;
                                    else jc0 += 1.f;
                                }
                            }
#pragma unroll
                            for (int o = 0; o < NO; ++o) {
                                // exact values: the j side gets them unscaled (no eps folding here)
                                jv[o] = f2add(jv[o], f2p(ja[o] / fscale[o], jbv[o] / fscale[o]));
                                double v = vi[o];
                                v += __shfl_xor_sync(0xffffffffu, v, 1);
                                v += __shfl_xor_sync(0xffffffffu, v, 2);
                                if (jq == 0 && li < np) S.acc[li][o] += v;
                            }
                            ci += __shfl_xor_sync(0xffffffffu, ci, 1);
                            ci += __shfl_xor_sync(0xffffffffu, ci, 2);
                            if (jq == 0 && li < np) S.cnt[li] += ci;
                            __syncwarp();
                        }
                    } else {
                        // the lane's staged j pair record and thresholds
                        const ulonglong2* pb = reinterpret_cast<const ulonglong2*>(S.sj + (e * 4 + jq) * (HL ? 12 : 8));
                        const ulonglong2 P0 = pb[0], P1 = pb[1];
                        ulonglong2 P2 = {0, 0};
                        if (HL) P2 = pb[2];
                        const float2 JL = S.jlo[e * 4 + jq], JH = S.jhi[e * 4 + jq];
                        for (uint32_t bits = m; bits; bits &= bits - 1) {
                            const uint32_t b = __ffs(bits) - 1;
                            const uint32_t li = b * 8 + il;
                            const uint64_t i = p0 + li;
                            const bool act = li < np;
                            const float lo_i = S.ilo[li], hi_i = S.ihi[li];
                            const float fxi = S.ix[li], fyi = S.iy[li], fzi = S.iz[li];
                            f2 dx = f2sub(f2p(fxi, fxi), P0.x), dy = f2sub(f2p(fyi, fyi), P0.y), dz = f2sub(f2p(fzi, fzi), P1.x);
                            if (HL) {
                                const float lxi = S.ilx[li], lyi = S.ily[li], lzi = S.ilz[li];
                                dx = f2add(dx, f2sub(f2p(lxi, lxi), P1.y));
                                dy = f2add(dy, f2sub(f2p(lyi, lyi), P2.x));
                                dz = f2add(dz, f2sub(f2p(lzi, lzi), P2.y));
                            }
                            float d2a, d2b;
                            f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                            // slots that are not evaluated: out of the SC / i == j / mirrored (j <= i)
                            if (!act || (selfe && ja_g <= i)) d2a = kFar;
                            if (!act || CJ == 4 || (selfe && jb_g <= i)) d2b = kFar;
                            const float La = fmaxf(lo_i, JL.x), Lb = fmaxf(lo_i, JL.y);
                            const float Ha = fmaxf(hi_i, JH.x), Hb = fmaxf(hi_i, JH.y);
                            float ma = fset_lt(d2a, La), mb = fset_lt(d2b, Lb);
                            const bool sa = (d2a <= Ha) & ((LJ & (d2a < close2)) | !(d2a < La));
                            const bool sb = (d2b <= Hb) & ((LJ & (d2b < close2)) | !(d2b < Lb));
                            // regular slots: fp32 values
                            f2 vals[4] = {0, 0, 0, 0};
                            const f2 m2 = f2p(sa ? 0.f : ma, sb ? 0.f : mb);
                            if (K == SFCNL_KERNEL_DENSITY) {
                                const float ih = S.iinvh[li];
                                const f2 q = f2mul(f2p(sqrt_ftz(d2a), sqrt_ftz(d2b)), f2p(ih, ih));
                                float q0, q1;
                                f2u(q, q0, q1);
                                const f2 tt = f2p(fmaxf(1.f - q0, 0.f), fmaxf(1.f - q1, 0.f));
                                const f2 uu = f2p(fmaxf(0.5f - q0, 0.f), fmaxf(0.5f - q1, 0.f));
                                const f2 tt2 = f2mul(tt, tt), uu2 = f2mul(uu, uu);
                                const f2 t3 = f2mul(tt2, tt), u3 = f2mul(uu2, uu);
                                const f2 wv = f2fma(f2p(-4.f, -4.f), u3, t3);  // W / (2 sigma)
                                float pma, pmb;
                                if constexpr (HL) {
                                    const float2 mm = S.sm[e * 4 + jq];
                                    pma = mm.x, pmb = mm.y;
                                } else {
                                    f2u(P1.y, pma, pmb);
                                }
                                const float sgi = 2.f * S.iscale[li];
                                const f2 mw = f2mul(f2p(pma * sgi, pmb * sgi), m2);
                                vals[0] = f2mul(mw, wv);
                                // |dW/dq| <= 2 sigma 3 (t^2 + 4 u^2): the bound is 3 dq sum of this channel
                                vals[1] = f2mul(mw, f2fma(f2p(4.f, 4.f), uu2, tt2));
                            } else if (LJ) {
                                const f2 inv2 = f2mul(f2p(rcp_ftz(d2a), rcp_ftz(d2b)), m2);
                                const f2 s2 = f2mul(f2p(sig2, sig2), inv2);
                                const f2 s6 = f2mul(f2mul(s2, s2), s2);
                                f2 cf = f2mul(inv2, f2mul(s6, f2fma(f2p(2.f, 2.f), s6, f2p(-1.f, -1.f))));
                                f2 ee = f2fma(s6, s6, f2mul(s6, f2p(-1.f, -1.f)));
                                if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                    cf = f2mul(cf, f2p(float(eps24d), float(eps24d)));
                                    ee = f2mul(ee, f2p(float(eps4d), float(eps4d)));
                                    const float qi = float(A.ck * A.q[i]);
                                    const float qa = (ma != 0.f && !sa) ? qi * float(A.q[ja_g]) : 0.f;
                                    const float qb = (CJ == 8 && mb != 0.f && !sb) ? qi * float(A.q[jb_g]) : 0.f;
                                    float ra, rb;
                                    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(d2a));
                                    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(d2b));
                                    const f2 qr = f2mul(f2p(qa, qb), f2p(ra, rb));
                                    ee = f2add(ee, qr);
                                    cf = f2fma(qr, inv2, cf);
                                }
                                vals[0] = f2mul(cf, dx), vals[1] = f2mul(cf, dy), vals[2] = f2mul(cf, dz), vals[3] = ee;
                            }
                            float cnt_a = sa ? 0.f : ma, cnt_b = sb ? 0.f : mb;
                            {  // special slots are deferred to the end of the chunk (no fp64 / calls here)
                                const unsigned ba = __ballot_sync(0xffffffffu, sa), bq = __ballot_sync(0xffffffffu, sb);
                                if (ba | bq) {
                                    const uint32_t item = e | (b << 5) | (lane << 8);
                                    if (sa) sq[qn + __popc(ba & lt_mask)] = item | (uint32_t(d2a < La) << 14);
                                    if (sb) sq[qn + __popc(ba) + __popc(bq & lt_mask)] = item | (1u << 13) | (uint32_t(d2b < Lb) << 14);
                                    qn += __popc(ba) + __popc(bq);
                                }
                            }
                            // i side: the two slots, then the four j-quarter lanes; fp64 sums in smem
#pragma unroll
                            for (int o = 0; o < NE; ++o) {
                                float a, c;
                                f2u(vals[o], a, c);
                                if (act) S.ip[li][jq][o] += a + c;
                                // j side: signed (odd outputs negated), over the bits of the entry
                                jv[o] = (NO == 4 && o < 3) ? f2sub(jv[o], vals[o]) : f2add(jv[o], vals[o]);
                            }
                            if (act) S.ipc[li][jq] += cnt_a + cnt_b;
                            jc0 += cnt_a, jc1 += cnt_b;
                        }
                    }
                    // j side of the entry: reduce over the eight i lanes, write [entry][j][o]
#pragma unroll
                    for (int o = 0; o < NE; ++o) {
                        float a, c;
                        f2u(jv[o], a, c);
#pragma unroll
                        for (int s = 4; s < 32; s <<= 1) a += __shfl_xor_sync(0xffffffffu, a, s), c += __shfl_xor_sync(0xffffffffu, c, s);
                        if (il == 0) {
                            S.jside[e][jq][o] = a;
                            if (CJ == 8) S.jside[e][jq + 4][o] = c;
                        }
                    }
#pragma unroll
                    for (int s = 4; s < 32; s <<= 1) jc0 += __shfl_xor_sync(0xffffffffu, jc0, s), jc1 += __shfl_xor_sync(0xffffffffu, jc1, s);
                    if (il == 0) {
                        S.jsc[e][jq] = uint32_t(jc0);
                        if (CJ == 8) S.jsc[e][jq + 4] = uint32_t(jc1);
                    }
                }
                __syncwarp();
                // deferred special slots: the reference predicate / fp64 kernel (LJ pairs known
                // to be in range: fp64 from the staged hi/lo), both sides
                for (uint32_t k = lane; k < qn; k += 32) {
                    const uint32_t it = sq[k];
                    const uint32_t e = it & 31u, b = (it >> 5) & 7u, ln = (it >> 8) & 31u, sl = (it >> 13) & 1u;
                    const bool inr = (it >> 14) & 1u;
                    const uint32_t li = b * 8 + (ln >> 2), q = ln & 3u, jj = q + 4 * sl;
                    const uint64_t i = p0 + li, j = uint64_t(S.idx[h0 + e]) * CJ + jj;
                    if (j >= A.n) continue;
                    double v[4];
                    int rc = -2;
                    if constexpr (LJ) {
                        if (inr) {
                            const float* pj = S.sj + (e * 4 + q) * 12 + sl;
                            const double ddx = (double(S.ix[li]) - double(pj[0])) + (double(S.ilx[li]) - double(pj[6]));
                            const double ddy = (double(S.iy[li]) - double(pj[2])) + (double(S.ily[li]) - double(pj[8]));
                            const double ddz = (double(S.iz[li]) - double(pj[4])) + (double(S.ilz[li]) - double(pj[10]));
                            const double dd2 = ddx * ddx + ddy * ddy + ddz * ddz;
                            if (dd2 >= double(kLjTiny2) * sig2d) {
                                const double inv2 = 1.0 / dd2;
                                const double s2 = sig2d * inv2, s6 = s2 * s2 * s2;
                                double coef = eps24d * inv2 * s6 * (2.0 * s6 - 1.0);
                                double en = eps4d * s6 * (s6 - 1.0);
                                if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                    const double qq = A.ck * A.q[i] * A.q[j], ir = sqrt(inv2);
                                    en += qq * ir;
                                    coef += qq * ir * inv2;
                                }
                                v[0] = coef * ddx, v[1] = coef * ddy, v[2] = coef * ddz, v[3] = en;
                                rc = 1;
                            }
                        }
                    }
                    if (rc == -2) rc = sym_exact_slot<K>(A, i, j, v);
                    if (rc < 0) coincident = true;
                    if (rc <= 0) continue;
#pragma unroll
                    for (int o = 0; o < NO; ++o) {
                        atomicAdd(&S.acc[li][o], v[o]);
                        // fp64 straight to the j particle (close LJ pairs can exceed the fp32 range)
                        atomicAdd(jspec + j * NO + o, (NO == 4 && o < 3) ? -v[o] : v[o]);
                    }
                    atomicAdd(&S.cnt[li], 1u);
                    atomicAdd(&S.jsc[e][jj], 1u);
                }
                qn = 0;
                __syncwarp();  // special-slot atomics done
                // the chunk's i-side partials into the per-i fp64 sums (j-quarter order)
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const uint32_t k = lane + 32u * s;
#pragma unroll
                    for (int o = 0; o < NE; ++o) {
                        const float v = (S.ip[k][0][o] + S.ip[k][1][o]) + (S.ip[k][2][o] + S.ip[k][3][o]);
                        S.ip[k][0][o] = S.ip[k][1][o] = S.ip[k][2][o] = S.ip[k][3][o] = 0.f;
                        S.acc[k][o] += double(v) * double(fscale[o]);
                    }
                    S.cnt[k] += uint32_t((S.ipc[k][0] + S.ipc[k][1]) + (S.ipc[k][2] + S.ipc[k][3]));
                    S.ipc[k][0] = S.ipc[k][1] = S.ipc[k][2] = S.ipc[k][3] = 0.f;
                }
                __syncwarp();
                // the chunk's j side to global: jacc[entry][j][o] (eps factors applied)
                for (uint32_t k = lane; k < n * CJ; k += 32) {
                    const uint32_t e = k / CJ, jj = k % CJ;
                    const uint64_t g = gE0 + bb + h0 + e;
#pragma unroll
                    for (int o = 0; o < NE; ++o) jacc[(g * CJ + jj) * NE + o] = S.jside[e][jj][o] * fscale[o];
                    jcnt[g * CJ + jj] = S.jsc[e][jj];
                }
                __syncwarp();  // the chunk's staging is consumed
            }
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        __syncwarp();
        if (!bad) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const uint32_t k = lane + 32u * s;
                if (k < np) {
#pragma unroll
                    for (int o = 0; o < NO; ++o) A.out[o][p0 + k] = (K == SFCNL_KERNEL_COUNT) ? double(S.cnt[k]) : S.acc[k][o];
                    if (NE > NO) aux[p0 + k] = S.acc[k][NE - 1];
                    A.cnt[p0 + k] = S.cnt[k];
                }
            }
        }
        __syncwarp();
    }
}

// Adds, per particle, the j-side sums of every entry whose j-cluster holds it (entry order).
template <int K>
__global__ void k_sym_fgather(uint64_t n, uint32_t cj, const float* __restrict__ jacc, const uint32_t* __restrict__ jcnt,
                              const uint64_t* __restrict__ tstart, const uint32_t* __restrict__ tlist, double* o0,
                              double* o1, double* o2, double* o3, uint32_t* __restrict__ cnt, double* __restrict__ aux,
                              const double* __restrict__ jspec) {
    constexpr int NO = nout<K>();
    constexpr int NE = PsSmem<K>::NE;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = p / cj, lane = p % cj;
        double acc[4] = {0, 0, 0, 0};
        uint32_t k = 0;
        for (uint64_t t = tstart[c]; t < tstart[c + 1]; ++t) {
            const uint64_t g = tlist[t];
#pragma unroll
            for (int o = 0; o < NE; ++o) acc[o] += double(jacc[(g * cj + lane) * NE + o]);
            k += jcnt[g * cj + lane];
        }
        double* outs[4] = {o0, o1, o2, o3};
        if (K == SFCNL_KERNEL_COUNT) {
            o0[p] += double(k);
        } else {
#pragma unroll
            for (int o = 0; o < NO; ++o) outs[o][p] += acc[o] + jspec[p * NO + o];
        }
        if (NE > NO) aux[p] += acc[NE - 1];
        cnt[p] += k;
    }
}

// The mixed symmetric density's a-posteriori error bound: 3 dq sum_j w_ij (spline slope
// weights, both sides) + 8 ulp rho, dq = 6 ulp qs (hi + lo staging: fp32 arithmetic only).
// Counts the particles that might miss the 1e-5 bar (sparse, edge-dominated neighbourhoods).
__global__ void k_sym_check(uint64_t n, double qs, const double* __restrict__ rho, const double* __restrict__ aux,
                            unsigned long long* __restrict__ flagged) {
    const double dq = 3.5762786865234375e-07 * qs;
    unsigned c = 0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x)
        c += 3.0 * dq * aux[p] + 4.76837158203125e-07 * rho[p] > 1.0e-5 * rho[p];
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane_id() == 0 && c) atomicAdd(flagged, (unsigned long long)c);
}
