// Warp-per-super-cluster mixed-precision pass (precision 1, gather, ci == 8,
// cj in {4, 8}); included by pass.cu after pass_fast.cuh (shares its helpers).
//
// Replaces the per-SC entry loop of reduce<Real,K> (reduce.hpp:94-197) for the
// built-in kernels. Every warp is independent: it takes the next super-cluster
// (SC) from a global counter and runs the whole SC alone, so the kernel has no
// block barriers and no producer/consumer hand-over; the warps of an SM hide
// each other's load latency.
//
// Per SC (64 particles, 8 i-clusters b):
//  * i side: the 64 particles are made relative to the SC's first particle in
//    fp64 (per-particle minimum image), rounded to fp32 (hi, + lo for LJ) and
//    kept in the warp's shared-memory slice with r_i and the kernel constants.
//  * per codec block (w entries, decoded by the warp in order: block mask ballot,
//    nibble-count scans, difference scan -- codec::decode_into,
//    nibble_codec.cpp:136-178) and per 32 entries of it:
//      stage: every j particle once, SC-relative fp32 in the packed-pair layout
//             {x_a,x_b,y_a,y_b,z_a,z_b,p_a,p_b} per (entry, j-quarter), slots
//             a = q, b = q + 4, so a lane's two slots load as f32x2 pairs;
//      compute: for each i-cluster b, the entries whose mask has bit b
//             (ballot + ffs); lane = (i in cluster b) x (j quarter), two slots
//             per lane in FFMA2/FADD2/FMUL2; partial sums are reduced over the
//             four j-quarter lanes and added into per-i fp64 sums in shared
//             memory once per (block, b).
//  * cutoff decisions: fp32 with the guard band of pass.cu; band slots (and LJ
//    pairs closer than kLjClose * sigma, where fp32 could overflow) go through
//    the reference's fp64 predicate and kernel (rare_slot), so neighbor_count is
//    exact. SCs whose periodic images are ambiguous in the SC frame ("unsafe")
//    evaluate every slot that way.
constexpr int kPwWarps = 4;    // independent warps per CTA
constexpr int kPwChunk = 32;   // entries staged at a time
// LJ pairs with d2 < kLjClose2 * sigma^2 are evaluated in fp64 from the staged
// hi/lo coordinates (in registers): the energy (s6 - 1) and force (2 s6 - 1)
// factors cross zero at d = sigma and 2^(1/6) sigma, where an fp32 term keeps an
// absolute error of ~1e-6 * 4 s6 that the 1e-5 * sum_j |E_ij| bar cannot absorb,
// and fp32 (sigma/d)^12 overflows for d -> 0. Pairs closer than kLjTiny2 * sigma^2
// (coincidence range) take the reference's fp64 path (rare_slot).
constexpr float kLjClose2 = 1.5f;
constexpr float kLjTiny2 = 1e-6f;
#ifdef SFCNL_PW_TWO
constexpr bool kTwo = true;
#else
constexpr bool kTwo = false;
#endif
constexpr bool kTwoDensityOff = true;
constexpr bool kPwF32Acc = true;  // LJ: fp32 per-i sums across chunks, fp64 only at the end (-0.4 %)

template <int K>
struct alignas(16) PwSmem {
    static constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    static constexpr int NO = nout<K>();
    static constexpr int kMinBlocks = LJ ? 4 : 6;  // CTAs of 4 warps per SM (registers: 128 / 85)
    // per (entry, j-quarter): density/count 8 floats {x_a,x_b,y_a,y_b,z_a,z_b,m_a,m_b};
    // LJ 12 floats {x_a,x_b,y_a,y_b, z_a,z_b,lx_a,lx_b, ly_a,ly_b,lz_a,lz_b} (hi, then lo)
    float sj[kPwChunk * 4 * (LJ ? 12 : 8)];
    uint32_t idx[64];                     // decoded block
    float ix[64], iy[64], iz[64];
    float ilx[LJ ? 64 : 1], ily[LJ ? 64 : 1], ilz[LJ ? 64 : 1];
    double iscale[64]; // density: 8/(pi h^3) * 2 (the spline's factor 2 folded in)
    float iinvh[64];   // density: 1 / h_i
    double acc[64][NO];
    float accf[LJ ? 64 : 1][NO];  // LJ: fp32 sums of the per-(b, chunk) flushes (fp64 close pairs stay in acc)
    uint32_t cnt[64];
    float ilo[64], ihi[64];  // per-chunk cutoff thresholds with the guard band
};

template <int K>
constexpr size_t pw_smem() {
    return size_t(kPwWarps) * sizeof(PwSmem<K>);
}

template <int K, int CJ>
__global__ void __launch_bounds__(kPwWarps * 32, PwSmem<K>::kMinBlocks) k_pass_warp(const __grid_constant__ PassArgs A,
                                                             unsigned long long* __restrict__ work) {
    constexpr bool LJ = PwSmem<K>::LJ;
    constexpr int NO = nout<K>();
    extern __shared__ __align__(16) unsigned char dsm[];
    PwSmem<K>& S = reinterpret_cast<PwSmem<K>*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    const uint32_t il = lane >> 2, jq = lane & 3;
    // the lane's j-quarter base in the shared window, pinned in a register (an opaque
    // mov keeps the compiler from re-deriving (e * 4 + jq) * stride in the entry loop)
    uint32_t sjq;
    asm volatile("mov.b32 %0, %1;" : "=r"(sjq) : "r"(uint32_t(__cvta_generic_to_shared(S.sj + jq * (LJ ? 12 : 8)))));
    const uint32_t w = uint32_t(A.w);
    const float sig2 = float(A.sigma * A.sigma);
    const float eps24 = float(24.0 * A.eps), eps4 = float(4.0 * A.eps);
    const float close2 = A.lj_close2 * sig2;
    const double sig2d = A.sigma * A.sigma, eps24d = 24.0 * A.eps, eps4d = 4.0 * A.eps;

    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        const uint64_t sc = A.sc_begin + __shfl_sync(0xffffffffu, t, 0);
        if (sc >= A.num_sc) break;

        // ---- open the SC's slice (decode_entry_indices, neighbor_store.cpp:18-42)
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

        // ---- i side
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
            double r = -1.0, hk = 1.0;
            double qx = 0, qy = 0, qz = 0;
            if (k < np) {
                qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                hk = A.h[p0 + k];
                fx = float(qx), fy = float(qy), fz = float(qz);
                r = dmul(A.qs, hk);
                eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                er = fmaxf(er, float(r));
            }
            S.ix[k] = fx, S.iy[k] = fy, S.iz[k] = fz;
            if (LJ) S.ilx[k] = float(qx - double(fx)), S.ily[k] = float(qy - double(fy)), S.ilz[k] = float(qz - double(fz));
            if (K == SFCNL_KERNEL_DENSITY) S.iscale[k] = 2.0 * (8.0 / (kPi * hk * hk * hk)), S.iinvh[k] = float(1.0 / hk);
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                S.acc[k][o] = 0.0;
                if (LJ) S.accf[k][o] = 0.f;
            }
            S.cnt[k] = 0;
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
        // per-particle min-imaging against the SC origin is exact for every in-range
        // pair when max|rel_i| + max r < L/2 on each periodic axis
        const bool unsafe = (A.box.per[0] && double(eax) + double(er) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(er) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(er) >= 0.49 * A.box.len[2]);
        const float Ei = fmaxf(eax, fmaxf(eay, eaz));
        __syncwarp();

        bool coincident = false;
        float E_run = -1.f;  // running bound of the staged |coordinates| for the guard bands
        uint64_t pos = 0, running = 0;
        const uint32_t nicl = tmin<uint32_t>(8u, uint32_t((np + 7) / 8));
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
            if (A.g2l)  // domain decomposition: stored global ids -> local clusters (same lanes as the decode)
                for (uint32_t k = lane; k < len; k += 32) S.idx[k] = A.g2l[S.idx[k]];
            __syncwarp();
            for (uint32_t h0 = 0; h0 < len; h0 += kPwChunk) {
                const uint32_t n = tmin<uint32_t>(kPwChunk, len - h0);
                const bool have = lane < n;
                const uint32_t my_idx = have ? S.idx[h0 + lane] : 0u;
                const uint32_t my_msk = have ? uint32_t(rec[bb + h0 + lane]) : 0u;
                // ---- stage the chunk's j particles (8 per lane, 4 loads in flight each)
                float emax = 0.f;
                if (!unsafe) {
                    float* sj = S.sj;
#pragma unroll
                    for (int k0 = 0; k0 < 8; k0 += 4) {
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
                                if (LJ) lx = float(qx - double(fx)), ly = float(qy - double(fy)), lz = float(qz - double(fz));
                                emax = fmaxf(emax, fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))));
                            }
                            const uint32_t q = jj & 3, hb = (jj < 4 || CJ == 8) ? (jj >> 2) : 1u;
                            if (!(jj < 4 || CJ == 8)) fx = fy = fz = kFar, fm = 0.f, lx = ly = lz = 0.f;  // cj == 4: slot b is a far dummy
                            if (LJ) {
                                float* p = sj + (e * 4 + q) * 12 + hb;
                                p[0] = fx, p[2] = fy, p[4] = fz, p[6] = lx, p[8] = ly, p[10] = lz;
                            } else {
                                float* p = sj + (e * 4 + q) * 8 + hb;
                                p[0] = fx, p[2] = fy, p[4] = fz, p[6] = fm;
                            }
                        }
                    }
                }
                const float E = fmaxf(Ei, warp_fmax(emax));
                if (!unsafe && E > E_run) {  // per-i thresholds (guard band of pass.cu); the band only
                    E_run = fmaxf(E, E_run * 1.0625f);  // widens with E: recomputed when a chunk raises it
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
                const int self_lo = int(p0) - (CJ - 1);  // j-clusters overlapping [p0, p0 + 64)
                const int jf = int(my_idx) * CJ - self_lo;
                const unsigned selfm = __ballot_sync(0xffffffffu, have && jf >= 0 && jf < kSC + CJ - 1);
                __syncwarp();

                for (uint32_t b = 0; b < nicl; ++b) {
                    unsigned mine = __ballot_sync(0xffffffffu, (my_msk >> b) & 1u);
                    if (!mine) continue;
                    const int li = int(b * 8 + il);
                    const uint64_t i = p0 + uint64_t(li);
                    const bool active = uint32_t(li) < np;
                    uint32_t cnt = 0;
                    if (unsafe) {
                        const double r = active ? dmul(A.qs, A.h[i]) : -1.0;
                        const double r2 = dmul(r, r);
                        // every slot through the reference predicate + fp64 kernel
                        double* side = &S.acc[li][0];
                        while (mine) {
                            const uint32_t e = __ffs(mine) - 1;
                            mine &= mine - 1;
                            const uint64_t jb = uint64_t(__shfl_sync(0xffffffffu, my_idx, e)) * CJ;
                            if (!active) continue;
                            if (jb + jq < A.n) {
                                const int rc = rare_slot<K, false>(A, i, jb + jq, r2, side);
                                cnt += rc > 0, coincident |= rc < 0;
                            }
                            if (CJ == 8 && jb + jq + 4 < A.n) {
                                const int rc = rare_slot<K, false>(A, i, jb + jq + 4, r2, side);
                                cnt += rc > 0, coincident |= rc < 0;
                            }
                        }
                        cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
                        cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
                        __syncwarp();
                        if (jq == 0) S.cnt[li] += cnt;
                        __syncwarp();
                        continue;
                    }
                    const float lo = S.ilo[li], hi_t = S.ihi[li];
                    const float fxi = S.ix[li], fyi = S.iy[li], fzi = S.iz[li];
                    const f2 xi2 = f2p(fxi, fxi), yi2 = f2p(fyi, fyi), zi2 = f2p(fzi, fzi);
                    f2 lxi2 = 0, lyi2 = 0, lzi2 = 0;
                    if (LJ) {
                        lxi2 = f2p(S.ilx[li], S.ilx[li]), lyi2 = f2p(S.ily[li], S.ily[li]), lzi2 = f2p(S.ilz[li], S.ilz[li]);
                    }
                    float inv_h = 0.f;
                    if (K == SFCNL_KERNEL_DENSITY) inv_h = S.iinvh[li];
                    f2 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, cntf = 0;
                    double accd0 = 0.0, accd1 = 0.0, accd2 = 0.0, accd3 = 0.0;  // LJ close pairs (fp64)

                    struct Ld {
                        f2 dx, dy, dz;
                        float pma, pmb, d2a, d2b;
                    };
                    auto load = [&](uint32_t e) {
                        Ld L;
                        // one IMAD per entry: the lane's j-quarter base is fixed per warp
                        const uint32_t a = sjq + e * (4 * (LJ ? 12 : 8) * 4);
                        ulonglong2 P0, P1;
                        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(P0.x), "=l"(P0.y) : "r"(a));
                        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2 + 16];" : "=l"(P1.x), "=l"(P1.y) : "r"(a));
                        L.dx = f2sub(xi2, P0.x);
                        L.dy = f2sub(yi2, P0.y);
                        L.dz = f2sub(zi2, P1.x);
                        if (LJ) {
                            ulonglong2 P2;  // {ly, lz} pairs; lx pair is P1.y
                            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2 + 32];" : "=l"(P2.x), "=l"(P2.y) : "r"(a));
                            L.dx = f2add(L.dx, f2sub(lxi2, P1.y));
                            L.dy = f2add(L.dy, f2sub(lyi2, P2.x));
                            L.dz = f2add(L.dz, f2sub(lzi2, P2.y));
                            L.pma = L.pmb = 0.f;
                        } else {
                            f2u(P1.y, L.pma, L.pmb);
                        }
                        f2u(f2fma(L.dz, L.dz, f2fma(L.dy, L.dy, f2mul(L.dx, L.dx))), L.d2a, L.d2b);
                        return L;
                    };
                    // special slot (divergent, rare): an in-range LJ pair closer than
                    // kLjClose * sigma (fp64 from the staged hi/lo coordinates; coincidence
                    // range through the reference path) or a cutoff inside the guard band
                    // (the reference predicate and fp64 kernel decide)
                    auto special = [&](uint32_t e, int sl2, float d2) {
                        const uint64_t j = uint64_t(S.idx[h0 + e]) * CJ + jq + 4 * sl2;
                        if (j >= A.n) return;
                        if (LJ && d2 < lo) {
                            const float* pj = S.sj + (e * 4 + jq) * 12 + sl2;
                            const double dx = (double(S.ix[li]) - double(pj[0])) + (double(S.ilx[li]) - double(pj[6]));
                            const double dy = (double(S.iy[li]) - double(pj[2])) + (double(S.ily[li]) - double(pj[8]));
                            const double dz = (double(S.iz[li]) - double(pj[4])) + (double(S.ilz[li]) - double(pj[10]));
                            const double dd2 = dx * dx + dy * dy + dz * dz;
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
                                accd0 += coef * dx, accd1 += coef * dy, accd2 += coef * dz, accd3 += en;
                                ++cnt;
                                return;
                            }
                        }
                        const double r = dmul(A.qs, A.h[i]);
                        const int rc = rare_slot<K, false>(A, i, j, dmul(r, r), &S.acc[li][0]);
                        cnt += rc > 0, coincident |= rc < 0;
                    };
                    auto compute = [&](uint32_t e, const Ld& L, auto SELF) {
                        constexpr bool kSelf = decltype(SELF)::value;
                        float d2a = L.d2a, d2b = L.d2b;
                        if (kSelf) {  // i == j slots drop out
                            const int jl0 = int(__shfl_sync(0xffffffffu, my_idx, e)) * CJ - int(p0);
                            if (jl0 + int(jq) == li) d2a = kFar;
                            if (CJ == 8 && jl0 + int(jq) + 4 == li) d2b = kFar;
                        }
                        float ma = fset_lt(d2a, lo), mb = fset_lt(d2b, lo);
                        // special: inside the guard band [lo, hi], or (LJ) closer than close2
                        // (bitwise, branch-free predicate logic; close2 < lo in every practical case,
                        // and a close slot beyond lo is just routed to the reference path)
                        const bool sa = (d2a <= hi_t) & ((LJ & (d2a < close2)) | !(d2a < lo));
                        const bool sb = (d2b <= hi_t) & ((LJ & (d2b < close2)) | !(d2b < lo));
                        if (sa | sb) {
                            if (sa) special(e, 0, d2a), ma = 0.f;
                            if (sb) special(e, 1, d2b), mb = 0.f;
                        }
                        const f2 m2 = f2p(ma, mb);
                        cntf = f2add(cntf, m2);
                        if (K == SFCNL_KERNEL_DENSITY) {
                            // W(q)/(2 sigma) = max(1-q,0)^3 - 4 max(1/2-q,0)^3
                            // max(1 - q, 0), max(1/2 - q, 0) as saturated fmas (q >= 0)
                            const float sa = sqrt_ftz(d2a), sb = sqrt_ftz(d2b);
                            const f2 t = f2p(__saturatef(fmaf(-sa, inv_h, 1.f)), __saturatef(fmaf(-sb, inv_h, 1.f)));
                            const f2 u = f2p(__saturatef(fmaf(-sa, inv_h, 0.5f)), __saturatef(fmaf(-sb, inv_h, 0.5f)));
                            const f2 t3 = f2mul(f2mul(t, t), t), u3 = f2mul(f2mul(u, u), u);
                            const f2 wv = f2fma(f2p(-4.f, -4.f), u3, t3);
                            acc0 = f2fma(f2mul(f2p(L.pma, L.pmb), m2), wv, acc0);
                        } else if (LJ) {
                            // m2 = 0 for out-of-range / special slots; d2 >= close2 > 0 here, so rcp is finite
                            const f2 inv2 = f2mul(f2p(rcp_ftz(d2a), rcp_ftz(d2b)), m2);
                            const f2 s2 = f2mul(f2p(A.sig2f, A.sig2f), inv2);
                            const f2 s6 = f2mul(f2mul(s2, s2), s2);
                            // 24 eps / 4 eps are applied at the flush (K == LJ)
                            // t = s6 - 1 (exact for s6 in [1/2, 2], where the factors cross zero),
                            // 2 s6 - 1 = s6 + t: one instruction less than the fma/mul forms
                            const f2 t = f2add(s6, f2p(-1.f, -1.f));
                            f2 cf = f2mul(f2mul(s6, inv2), f2add(s6, t));
                            f2 ee = f2mul(s6, t);  // LJ: fused into the energy sum below
                            if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                cf = f2mul(cf, f2p(eps24, eps24));
                                ee = f2mul(ee, f2p(eps4, eps4));
                                const uint64_t jb = uint64_t(S.idx[h0 + e]) * CJ;
                                const float qi = float(A.ck * A.q[i]);
                                const float qa = ma != 0.f ? qi * float(A.q[jb + jq]) : 0.f;
                                const float qb = (CJ == 8 && mb != 0.f) ? qi * float(A.q[jb + jq + 4]) : 0.f;
                                float ra, rb;
                                asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(d2a));
                                asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(d2b));
                                const f2 qr = f2mul(f2p(qa, qb), f2p(ra, rb));
                                ee = f2add(ee, qr);
                                cf = f2fma(qr, inv2, cf);
                            }
                            acc0 = f2fma(cf, L.dx, acc0);
                            acc1 = f2fma(cf, L.dy, acc1);
                            acc2 = f2fma(cf, L.dz, acc2);
                            if (K == SFCNL_KERNEL_LJ) acc3 = f2fma(s6, t, acc3);  // energy s6 (s6 - 1), fused
                            else acc3 = f2add(acc3, ee);
                        }
                    };
                    unsigned ms = mine & selfm;
                    mine &= ~selfm;
                    while (mine) {
                        // highest entry first: FLO gives it directly (ffs needs a bit reversal),
                        // BMSK keeps the bits below it (no shifted-one constant to hold)
                        uint32_t e1, below;
                        asm("bfind.u32 %0, %1;" : "=r"(e1) : "r"(mine));
                        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(e1));
                        mine &= below;
                        if (kTwo && (LJ || !kTwoDensityOff) && mine) {  // two entries in flight
                            const uint32_t e2 = __ffs(mine) - 1;
                            mine &= mine - 1;
                            const Ld L1 = load(e1), L2 = load(e2);
                            compute(e1, L1, BoolC<false>());
                            compute(e2, L2, BoolC<false>());
                        } else {
                            compute(e1, load(e1), BoolC<false>());
                        }
                    }
                    while (ms) {
                        const uint32_t e = __ffs(ms) - 1;
                        ms &= ms - 1;
                        compute(e, load(e), BoolC<true>());
                    }
                    // flush: pair halves and the four j-quarter lanes of each i in fp32 (<= 2 x 64
                    // terms per lane), added to the per-i fp64 sums; fp64 close-pair sums separately
                    double tot[NO];
                    float totf[NO];
                    bool close_any = false;
                    const f2 accs[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
                    for (int o = 0; o < NO; ++o) {
                        float a, c;
                        f2u(accs[o], a, c);
                        float v = a + c;
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        const double sc_o = K == SFCNL_KERNEL_LJ ? (o < 3 ? eps24d : eps4d) : 1.0;
                        totf[o] = v;
                        tot[o] = kPwF32Acc && LJ ? 0.0 : double(v) * sc_o;
                    }
                    if (LJ && __any_sync(0xffffffffu, accd0 != 0.0 || accd1 != 0.0 || accd2 != 0.0 || accd3 != 0.0)) {
                        double accds[4] = {accd0, accd1, accd2, accd3};
                        close_any = true;
#pragma unroll
                        for (int o = 0; o < NO; ++o) {
                            double v = accds[o];
                            v += __shfl_xor_sync(0xffffffffu, v, 1);
                            v += __shfl_xor_sync(0xffffffffu, v, 2);
                            tot[o] += v;
                        }
                    }
                    {
                        float c0, c1;
                        f2u(cntf, c0, c1);
                        cnt += uint32_t(c0 + c1);
                    }
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
                    __syncwarp();  // rare-slot side sums of this b are complete
                    if (jq == 0 && active) {
                        if (K == SFCNL_KERNEL_DENSITY) {
                            S.acc[li][0] += S.iscale[li] * tot[0];
                        } else if (LJ) {
                            // fp32 per i across the SC's chunks (<= ~8 more roundings of partial sums),
                            // the fp64 close-pair sums into the fp64 side sums
#pragma unroll
                            for (int o = 0; o < NO; ++o) S.accf[li][o] += totf[o];
                            if (close_any) {
#pragma unroll
                                for (int o = 0; o < NO; ++o) S.acc[li][o] += tot[o];
                            }
                        }
                        S.cnt[li] += cnt;
                    }
                    __syncwarp();
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
                    const uint64_t i = p0 + k;
                    if (K == SFCNL_KERNEL_COUNT) {
                        A.out[0][i] = double(S.cnt[k]);
                    } else {
#pragma unroll
                        for (int o = 0; o < NO; ++o) {
                            double v = S.acc[k][o];
                            if (LJ && kPwF32Acc) v += double(S.accf[k][o]) * (K == SFCNL_KERNEL_LJ ? (o < 3 ? eps24d : eps4d) : 1.0);
                            A.out[o][i] = v;
                        }
                    }
                    A.cnt[i] = S.cnt[k];
                }
            }
        }
        __syncwarp();  // the warp's slice is reused by its next SC
    }
}
