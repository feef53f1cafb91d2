// Bit-exact fp64 pass (precision 0) for gather stores with ci == 8, cj in {4, 8};
// included by pass.cu after pass_fast.cuh (shares its helpers).
//
// Same values as k_pass_exact, and so as reduce<double> (reduce.hpp:151-197): every
// in-range pair is evaluated with the reference's round-to-nearest fp64 expressions
// (builtin_kernels.hpp:12-95) and added to its target's sum in the reference order
// (entries ascending, j ascending within the entry). What changes is where the fp64
// work runs: only ~1/3 of a cluster pair's slots are in range, and a thread-per-target
// loop pays the division / square root of the kernel on every slot any lane of the
// warp has in range. Here, warp per super-cluster (SC), per chunk of 32 entries:
//  1. stage the chunk's j particles once: fp64 (x, y, z, payload) for the evaluation,
//     SC-relative fp32 for the classification;
//  2. classify, lane = (target i of cluster b) x (every 4th entry of b): a slot whose
//     fp32 squared distance is <= r_i^2 + guard band (pass.cu's bound: a superset of the
//     in-range slots) sets a bit of the 8-bit hit mask of (i, entry);
//  3. evaluate: the targets with hits in the chunk are jobs handed out to lanes on
//     demand; a lane walks its target's hit bits in entry / j order, recomputes the
//     exact periodic_delta d2, skips the slot when d2 > r_i^2, else adds the kernel
//     value to the target's fp64 sum (shared memory, carried across chunks).
// SCs whose periodic images are ambiguous in the SC frame ("unsafe") mark every slot.
constexpr int kPxWarps = 4;
#ifndef SFCNL_PX_SLOTS
#define SFCNL_PX_SLOTS 4
#endif
constexpr int kPxSlots = SFCNL_PX_SLOTS;  // marked slots evaluated per step of a lane

template <int K>
struct alignas(16) PxSmem {
    static constexpr int NO = nout<K>();
    static constexpr bool kPay = K == SFCNL_KERNEL_DENSITY || K == SFCNL_KERNEL_LJ_COULOMB;
    double jx[256], jy[256], jz[256];  // [entry * 8 + jj] staged fp64 positions
    double jp[kPay ? 256 : 1];         // payload: m (density) or q (LJ+Coulomb)
    float fx[256], fy[256], fz[256];   // SC-relative fp32 (far away: invalid slot)
    alignas(16) uint8_t hm[64][32];    // hit masks [target][entry]
    uint32_t nz[64];                   // entries of the chunk with hits, per target
    uint32_t hc[64];                   // marked slots of the chunk, per target (job length)
    uint32_t jobs[64];                 // targets with hits, longest first
    double tx[64], ty[64], tz[64];     // targets: fp64 position, h, r^2 and the hoisted factor
    double th[64], tr2[64], tk[64];    // (8 / (pi h^3) for density, ck * q_i for Coulomb)
    uint32_t idx[64];                  // decoded codec block
    float fxi[64], fyi[64], fzi[64];   // targets, SC-relative fp32
    float ihi[64];                     // classification thresholds (current chunk)
    double acc[64][NO];
    uint32_t cnt[64];
};

template <int K>
constexpr size_t px_smem() {
    return size_t(kPxWarps) * sizeof(PxSmem<K>);
}

// Kernel value of one in-range pair, the expression chain of eval_exact with the
// per-target factors hoisted (they depend on h_i / q_i only, so the values are equal):
// sg = 8 / (pi h^3) (density), qci = ck * q_i (Coulomb). Returns 1 for a coincident LJ pair.
template <int K>
__device__ __forceinline__ int eval_x64(const PassArgs& A, double d2, double dx, double dy, double dz, double hi,
                                        double sg, double pj, double qci, double v[4]) {
    if (K == SFCNL_KERNEL_COUNT) {
        v[0] = 1.0;
    } else if (K == SFCNL_KERNEL_DENSITY) {
        const double r = __dsqrt_rn(d2);
        const double q = ddiv(r, hi);
        double w = 0.0;
        if (!(q > 1.0)) {
            if (q <= 0.5) {
                w = dmul(sg, dadd(1.0, dmul(dmul(dmul(6.0, q), q), dsub(q, 1.0))));
            } else {
                const double t = dsub(1.0, q);
                w = dmul(dmul(dmul(dmul(sg, 2.0), t), t), t);
            }
        }
        v[0] = dmul(pj, w);
    } else {
        if (d2 == 0.0) return 1;
        const double inv2 = ddiv(1.0, d2);
        const double s2 = dmul(dmul(A.sigma, A.sigma), inv2);
        const double s6 = dmul(dmul(s2, s2), s2);
        double coef = dmul(dmul(dmul(24.0, A.eps), inv2), dsub(dmul(dmul(2.0, s6), s6), s6));
        double en = dmul(dmul(4.0, A.eps), dsub(dmul(s6, s6), s6));
        if (K == SFCNL_KERNEL_LJ_COULOMB) {
            const double qq = dmul(qci, pj);
            const double inv_r = __dsqrt_rn(inv2);
            en = dadd(en, dmul(qq, inv_r));
            coef = dadd(coef, dmul(dmul(qq, inv_r), inv2));
        }
        v[0] = dmul(coef, dx), v[1] = dmul(coef, dy), v[2] = dmul(coef, dz), v[3] = en;
    }
    return 0;
}

template <int K, int CJ>
__global__ void __launch_bounds__(kPxWarps * 32, 3) k_pass_x64(const __grid_constant__ PassArgs A,
                                                           unsigned long long* __restrict__ work) {
    constexpr int NO = nout<K>();
    constexpr bool kPay = PxSmem<K>::kPay;
    extern __shared__ __align__(16) unsigned char dsm[];
    PxSmem<K>& S = reinterpret_cast<PxSmem<K>*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    const unsigned ltmask = (1u << lane) - 1u;
    const uint32_t il = lane >> 2, q4 = lane & 3;
    const uint32_t w = uint32_t(A.w);
    const double* pay = K == SFCNL_KERNEL_DENSITY ? A.m : A.q;

    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        const uint64_t sc = A.sc_begin + __shfl_sync(0xffffffffu, t, 0);
        if (sc >= A.num_sc) break;

        // ---- the SC's slice (decode_entry_indices, neighbor_store.cpp:18-42)
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

        // ---- targets: SC-relative fp32 positions, zeroed sums
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
            float fx = kFar, fy = kFar, fz = kFar;
            if (k < np) {
                const double qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                fx = float(qx), fy = float(qy), fz = float(qz);
                eax = fmaxf(eax, fabsf(fx)), eay = fmaxf(eay, fabsf(fy)), eaz = fmaxf(eaz, fabsf(fz));
                er = fmaxf(er, float(dmul(A.qs, A.h[p0 + k])));
            }
            S.fxi[k] = fx, S.fyi[k] = fy, S.fzi[k] = fz;
            if (k < np) {
                const double hh = A.h[p0 + k], r = dmul(A.qs, hh);
                S.tx[k] = A.x[p0 + k], S.ty[k] = A.y[p0 + k], S.tz[k] = A.z[p0 + k];
                S.th[k] = hh, S.tr2[k] = dmul(r, r);
                if (K == SFCNL_KERNEL_DENSITY) S.tk[k] = ddiv(8.0, dmul(dmul(dmul(kPi, hh), hh), hh));
                if (K == SFCNL_KERNEL_LJ_COULOMB) S.tk[k] = dmul(A.ck, A.q[p0 + k]);
            }
#pragma unroll
            for (int o = 0; o < NO; ++o) S.acc[k][o] = 0.0;
            S.cnt[k] = 0;
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
        // per-particle minimum images against the SC origin are exact for every
        // in-range pair when max|rel_i| + max r < L/2 on each periodic axis (with margin)
        const bool unsafe = (A.box.per[0] && double(eax) + double(er) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(er) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(er) >= 0.49 * A.box.len[2]);
        const float Ei = fmaxf(eax, fmaxf(eay, eaz));
        const uint32_t nicl = tmin<uint32_t>(8u, uint32_t((np + 7) / 8));
        bool coincident = false;
        __syncwarp();

        uint64_t pos = 0, running = 0;
        for (uint32_t bb = 0; !bad && bb < count; bb += w) {
            const uint32_t len = tmin<uint32_t>(w, count - bb);
            // ---- decode one codec block into S.idx[0, len)
            if (A.dec) {  // decoded once per store (k_decode_store)
                const uint32_t* src = A.dec + A.dec_base[sc - A.sc_begin] + bb;
                for (uint32_t k = lane; k < len; k += 32) S.idx[k] = src[k];
            } else if (A.compress) {
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
            if (A.g2l)
                for (uint32_t k = lane; k < len; k += 32) S.idx[k] = A.g2l[S.idx[k]];
            __syncwarp();
            for (uint32_t h0 = 0; h0 < len; h0 += 32) {
                const uint32_t n = tmin<uint32_t>(32, len - h0);
                const uint32_t my_msk = lane < n ? uint32_t(rec[bb + h0 + lane]) : 0u;

                // ---- 1. stage (lane = particle of entry e = 4u + lane / 8)
                float emax = 0.f;
#pragma unroll
                for (int u0 = 0; u0 < 8; u0 += 4) {
                    double vx[4], vy[4], vz[4], vp[4];
                    bool val[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t e = uint32_t(u0 + u) * 4 + (lane >> 3), jj = lane & 7;
                        const uint64_t j = uint64_t(S.idx[h0 + (e < n ? e : 0)]) * CJ + jj;
                        val[u] = e < n && jj < uint32_t(CJ) && j < A.n;
                        vx[u] = vy[u] = vz[u] = vp[u] = 0.0;
                        if (val[u]) {
                            vx[u] = A.x[j], vy[u] = A.y[j], vz[u] = A.z[j];
                            if (kPay) vp[u] = pay[j];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t e = uint32_t(u0 + u) * 4 + (lane >> 3), jj = lane & 7;
                        const uint32_t sl = e * 8 + jj;
                        float fx = kFar, fy = kFar, fz = kFar;
                        if (val[u]) {
                            fx = float(rel(vx[u], ox, 0)), fy = float(rel(vy[u], oy, 1)), fz = float(rel(vz[u], oz, 2));
                            emax = fmaxf(emax, fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))));
                        }
                        S.jx[sl] = vx[u], S.jy[sl] = vy[u], S.jz[sl] = vz[u];
                        if (kPay) S.jp[sl] = vp[u];
                        S.fx[sl] = fx, S.fy[sl] = fy, S.fz[sl] = fz;
                    }
                }
                // classification thresholds r_i^2 + guard band (pass.cu's bound for
                // coordinates rounded to fp32, each with error <= 2^-24 |coordinate|)
                const double E = double(fmaxf(Ei, warp_fmax(emax)));
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const uint32_t k = lane + 32u * s;
                    float hi = -1.f;
                    if (k < np) {
                        const double r = dmul(A.qs, A.h[p0 + k]), r2 = dmul(r, r);
                        const double ex = 1.1920928955078125e-07 * E + 5.9604644775390625e-08 * r;
                        hi = __double2float_ru(r2 + 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300);
                    }
                    S.ihi[k] = hi;
                }
                {
                    uint4* z = reinterpret_cast<uint4*>(&S.hm[0][0]);
#pragma unroll
                    for (int k = 0; k < 4; ++k) z[lane + 32 * k] = make_uint4(0u, 0u, 0u, 0u);
                }
                __syncwarp();

                // ---- 2. classify: lane = (target il of cluster b, every 4th entry of b)
                for (uint32_t b = 0; b < nicl; ++b) {
                    const unsigned mb = __ballot_sync(0xffffffffu, (my_msk >> b) & 1u);
                    if (!mb) {
                        if (q4 == 0) S.nz[b * 8 + il] = 0, S.hc[b * 8 + il] = 0;
                        continue;
                    }
                    const uint32_t i = b * 8 + il;
                    const bool active = i < np;
                    unsigned m = mb;
                    for (uint32_t k = 0; k < q4; ++k) m &= m - 1;
                    uint32_t nzp = 0, hcp = 0;
                    const float hi = S.ihi[i];
                    const f2 xi2 = f2p(S.fxi[i], S.fxi[i]), yi2 = f2p(S.fyi[i], S.fyi[i]), zi2 = f2p(S.fzi[i], S.fzi[i]);
                    const int self = int(p0) + int(i);
                    while (active && m) {
                        const uint32_t e = __ffs(m) - 1;
#pragma unroll
                        for (int k = 0; k < 4; ++k) m &= m - 1;
                        const int jg0 = int(S.idx[h0 + e]) * CJ;
                        uint32_t hmask = 0;
                        if (unsafe) {
                            hmask = CJ == 8 ? 0xffu : 0x0fu;
                        } else {
                            const f2* px = reinterpret_cast<const f2*>(&S.fx[e * 8]);
                            const f2* py = reinterpret_cast<const f2*>(&S.fy[e * 8]);
                            const f2* pz = reinterpret_cast<const f2*>(&S.fz[e * 8]);
#pragma unroll
                            for (int p = 0; p < CJ / 2; ++p) {
                                const f2 dx = f2sub(xi2, px[p]), dy = f2sub(yi2, py[p]), dz = f2sub(zi2, pz[p]);
                                float d2a, d2b;
                                f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                                hmask |= (d2a <= hi ? 1u : 0u) << (2 * p);
                                hmask |= (d2b <= hi ? 1u : 0u) << (2 * p + 1);
                            }
                        }
                        // i == j drops out; slots past the last particle never count
                        const int sj = self - jg0;
                        if (sj >= 0 && sj < CJ) hmask &= ~(1u << sj);
                        if (uint64_t(jg0) + CJ > A.n) hmask &= (1u << uint32_t(A.n - uint64_t(jg0))) - 1u;
                        if (hmask) S.hm[i][e] = uint8_t(hmask), nzp |= 1u << e, hcp += __popc(hmask);
                    }
                    nzp |= __shfl_xor_sync(0xffffffffu, nzp, 1);
                    nzp |= __shfl_xor_sync(0xffffffffu, nzp, 2);
                    hcp += __shfl_xor_sync(0xffffffffu, hcp, 1);
                    hcp += __shfl_xor_sync(0xffffffffu, hcp, 2);
                    if (q4 == 0) S.nz[i] = nzp, S.hc[i] = hcp;
                }
                for (uint32_t b = nicl; b < 8; ++b)
                    if (q4 == 0) S.nz[b * 8 + il] = 0, S.hc[b * 8 + il] = 0;
                __syncwarp();

                // ---- 3. evaluate: jobs = targets with hits, handed out on demand, longest
                // first (lanes that finish early take the short ones)
                uint32_t njobs = 0;
                {
                    const uint32_t c0 = S.hc[lane], c1 = S.hc[lane + 32];
                    uint32_t r0 = 0, r1 = 0;
                    for (uint32_t m = 0; m < 64; ++m) {
                        const uint32_t c = S.hc[m];
                        r0 += (c > c0) | ((c == c0) & (m < lane));
                        r1 += (c > c1) | ((c == c1) & (m < lane + 32));
                    }
                    if (c0) S.jobs[r0] = lane;
                    if (c1) S.jobs[r1] = lane + 32;
                    njobs = __popc(__ballot_sync(0xffffffffu, c0 != 0)) + __popc(__ballot_sync(0xffffffffu, c1 != 0));
                }
                __syncwarp();
                int job = -1;
                uint32_t jnz = 0, jm = 0, je = 0, jc = 0;
                double xi = 0, yi = 0, zi = 0, r2 = 0, hh = 0, sg = 0, qci = 0;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                uint32_t next = 0;
                for (;;) {
                    const bool need = jm == 0 && jnz == 0;
                    if (need && job >= 0) {
#pragma unroll
                        for (int o = 0; o < NO; ++o) S.acc[job][o] = acc[o];
                        S.cnt[job] = jc;
                        job = -1;
                    }
                    const unsigned nb = __ballot_sync(0xffffffffu, need);
                    if (need) {
                        const uint32_t k = next + __popc(nb & ltmask);
                        if (k < njobs) {
                            job = int(S.jobs[k]);
                            jnz = S.nz[job];
                            xi = S.tx[job], yi = S.ty[job], zi = S.tz[job], hh = S.th[job], r2 = S.tr2[job];
                            if (K == SFCNL_KERNEL_DENSITY) sg = S.tk[job];
                            if (K == SFCNL_KERNEL_LJ_COULOMB) qci = S.tk[job];
#pragma unroll
                            for (int o = 0; o < NO; ++o) acc[o] = S.acc[job][o];
                            jc = S.cnt[job];
                        }
                    }
                    next += __popc(nb);
                    if (!__any_sync(0xffffffffu, job >= 0)) break;
                    if (job < 0) continue;
                    // kPxSlots marked slots per step (independent fp64 chains), added in order
                    uint32_t sl[kPxSlots];
                    uint32_t nsl = 0;
#pragma unroll
                    for (int t = 0; t < kPxSlots; ++t) {
                        if (jm == 0 && jnz == 0) break;
                        if (jm == 0) {
                            je = __ffs(jnz) - 1;
                            jnz &= jnz - 1;
                            jm = S.hm[job][je];
                        }
                        sl[t] = je * 8 + (__ffs(jm) - 1);
                        jm &= jm - 1;
                        ++nsl;
                    }
#pragma unroll
                    for (int t = 1; t < kPxSlots; ++t)
                        if (uint32_t(t) >= nsl) sl[t] = sl[0];
                    double d2[kPxSlots], dx[kPxSlots], dy[kPxSlots], dz[kPxSlots], v[kPxSlots][4];
                    int bad2[kPxSlots];
#pragma unroll
                    for (int t = 0; t < kPxSlots; ++t) {
                        d2[t] = pair_d2_exact(xi, yi, zi, S.jx[sl[t]], S.jy[sl[t]], S.jz[sl[t]], A.box, &dx[t], &dy[t], &dz[t]);
                        bad2[t] = eval_x64<K>(A, d2[t], dx[t], dy[t], dz[t], hh, sg, kPay ? S.jp[sl[t]] : 0.0, qci, v[t]);
                    }
#pragma unroll
                    for (int t = 0; t < kPxSlots; ++t) {
                        if (uint32_t(t) >= nsl || d2[t] > r2) continue;
                        if (bad2[t]) {
                            coincident = true;
                            continue;
                        }
#pragma unroll
                        for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], v[t][o]);
                        ++jc;
                    }
                }
                __syncwarp();  // the chunk's staging and hit masks are consumed
            }
        }
        if (__any_sync(0xffffffffu, coincident) && lane == 0) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        __syncwarp();
        if (!bad) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const uint32_t k = lane + 32u * s;
                if (k < np) {
                    const uint64_t i = p0 + k;
#pragma unroll
                    for (int o = 0; o < NO; ++o) A.out[o][i] = S.acc[k][o];
                    A.cnt[i] = S.cnt[k];
                }
            }
        }
        __syncwarp();  // the warp's slice is reused by its next SC
    }
}
