// Item-parallel mixed-precision pass (precision 1, gather, ci == 8, cj in {4, 8});
// included by pass.cu after pass_fast.cuh (shares its helpers).
//
// Replaces the per-SC entry loop of reduce<Real,K> (reduce.hpp:94-197) for the
// built-in kernels. Warps are independent (no block barriers): a warp takes the
// next super-cluster (SC) from a global counter and runs it alone.
//
// Per SC: the 64 i particles are made relative to the SC's first particle (fp64,
// per-particle minimum image) and rounded to fp32. The entry list is decoded one
// codec block at a time by the warp (codec::decode_into, nibble_codec.cpp:136-178).
// Per 32 entries (a "chunk"):
//  * stage: every j particle once into shared memory in the SC frame, pair-packed
//    ([j pair p][entry e] float4s) -- from the cluster-frame copy for density/count
//    (frame.cu: one fp64 shift per entry + one fp32 add per coordinate), from fp64
//    as hi + lo fp32 for Lennard-Jones;
//  * items: every (i-cluster b, entry e) whose mask has bit b becomes one item,
//    listed b-major (non-self entries first, then entries overlapping the SC's own
//    particles, which need the i != j exclusion);
//  * rounds of 32 items, ONE ITEM PER LANE: the lane loads its entry's 8 j particles
//    into registers and evaluates all 8 x 8 slots (i outer, two j slots per FFMA2 /
//    FADD2 / FMUL2), with no ballots or shuffles in the slot loop;
//  * the per-(item, i) partial sums are reduced deterministically: written to
//    shared memory, then summed per i over the round's items of its i-cluster in
//    item order and added to per-i fp64 sums.
// Cutoff decisions: fp32 against per-i thresholds with the guard band of pass.cu
// (widened for the cluster-frame rounding); a row with a slot inside the band is
// re-examined and its band slots go through the reference fp64 predicate and kernel
// (rare_slot), so neighbor_count is exact. LJ pairs closer than kLjClose * sigma
// are evaluated in fp64 from the staged hi/lo coordinates (see pass_warp.cuh).
// SCs whose periodic images are ambiguous in the SC frame ("unsafe") evaluate every
// slot through rare_slot.
constexpr int kPiWarps = 4;
constexpr double kPiDensityDq = 2.0e-6;  // max staged-distance error / h of a density SC on the fp32 path

template <int K>
struct PiSmem {
    static constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    static constexpr int NO = nout<K>();
    float4 sa[4][32];           // {x_2p, x_2p+1, y_2p, y_2p+1}
    float4 sb[4][32];           // density/count {z, z', m, m'}; LJ {z, z', lx, lx'}
    float4 sc[LJ ? 4 : 1][32];  // LJ {ly, ly', lz, lz'}
    float4 ia[64];              // [ii*8 + b] {x, y, z, 1/h}
    float4 ib[64];              // [ii*8 + b] {lo, hi, lx, ly}
    float ic[64];               // [ii*8 + b] lz
    double ir[64];              // [i] r_i = query_scale * h_i (< 0: inactive)
    double iscale[K == SFCNL_KERNEL_DENSITY ? 64 : 1];  // [i] density: 2 * 8 / (pi h^3)
    double acc[64][NO];
    uint32_t cnt[64];
#ifndef SFCNL_PI_PAD
#define SFCNL_PI_PAD 1
#endif
    // per round: [row ii][output | count][lane]; rows padded so the per-i reduction (lanes
    // of one i-cluster read the same item column of 8 different rows) is conflict-free
    float part[8][NO + 1][32 + SFCNL_PI_PAD];
    uint32_t idx[64];
    uint8_t items[256];
};

template <int K>
constexpr size_t pi_smem() {
    return size_t(kPiWarps) * sizeof(PiSmem<K>);
}

__device__ __forceinline__ f2 f2lo(ulonglong2 v) { return v.x; }
__device__ __forceinline__ f2 f2hi(ulonglong2 v) { return v.y; }

// NM (density, query scale >= 1): a slot out of range has d2_f32 > hi = r^2 + guard with
// r = qs h >= h, so its fp32 q is >= 1 up to the sqrt / 1/h rounding (~4e-7, below the
// guard's relative margin) and W = max(1-q,0)^3 - 4 max(1/2-q,0)^3 is 0 -- no mask needed;
// a guard-band slot (decided by the fp64 path) keeps an fp32 W below (1e-6)^3 W(0).
#ifndef SFCNL_PI_NOMASK
#define SFCNL_PI_NOMASK 1
#endif
#ifndef SFCNL_PI_CTAS
#define SFCNL_PI_CTAS 5
#endif
template <int K, int CJ, bool NM = false>
__global__ void __launch_bounds__(kPiWarps * 32, PiSmem<K>::LJ ? 4 : SFCNL_PI_CTAS) k_pass_item(const __grid_constant__ PassArgs A,
                                                             unsigned long long* __restrict__ work) {
    constexpr bool LJ = PiSmem<K>::LJ;
    constexpr int NO = nout<K>();
    extern __shared__ __align__(16) unsigned char dsm[];
    PiSmem<K>& S = reinterpret_cast<PiSmem<K>*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    const unsigned ltmask = (1u << lane) - 1u;
    const uint32_t w = uint32_t(A.w);
    const float sig2 = float(A.sigma * A.sigma);
    const float eps24 = float(24.0 * A.eps), eps4 = float(4.0 * A.eps);
    const float close2 = A.lj_close2 * sig2;
    const double sig2d = A.sigma * A.sigma, eps24d = 24.0 * A.eps, eps4d = 4.0 * A.eps;
    // frame staging (density/count): max |offset| per axis of the cluster-frame copy
    float X = 0.f, Xax[3] = {0.f, 0.f, 0.f};
    if (!LJ) {
        for (int d = 0; d < 3; ++d) Xax[d] = __uint_as_float(A.frame_x[d]);
        X = fmaxf(Xax[0], fmaxf(Xax[1], Xax[2]));
    }

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
        float eax = 0.f, eay = 0.f, eaz = 0.f, er = 0.f, hmin = 3.0e38f;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const uint32_t k = lane + 32u * s;
            const uint32_t slot = (k & 7) * 8 + (k >> 3);
            float fx = 0.f, fy = 0.f, fz = 0.f;
            double r = -1.0, hk = 1.0, qx = 0, qy = 0, qz = 0;
            if (k < np) {
                qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                hk = A.h[p0 + k];
                fx = float(qx), fy = float(qy), fz = float(qz);
                r = dmul(A.qs, hk);
                eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                er = fmaxf(er, float(r));
                hmin = fminf(hmin, float(hk));
            }
            S.ia[slot] = make_float4(fx, fy, fz, float(1.0 / hk));
            if (LJ) {
                S.ib[slot].z = float(qx - double(fx)), S.ib[slot].w = float(qy - double(fy));
                S.ic[slot] = float(qz - double(fz));
            }
            S.ir[k] = r;
            if (K == SFCNL_KERNEL_DENSITY) S.iscale[k] = 2.0 * (8.0 / (kPi * hk * hk * hk));
#pragma unroll
            for (int o = 0; o < NO; ++o) S.acc[k][o] = 0.0;
            S.cnt[k] = 0;
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
        // per-particle / per-cluster images against the SC origin are exact for every
        // in-range pair when max|rel_i| + max r (+ X for the cluster frame) < 0.49 L
        const bool unsafe = (A.box.per[0] && double(eax) + double(er) + double(Xax[0]) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(er) + double(Xax[1]) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(er) + double(Xax[2]) >= 0.49 * A.box.len[2]);
        const float Ei = fmaxf(eax, fmaxf(eay, eaz));
        // W(q) near the support edge amplifies the distance error (|dW/dq| / W ~ 3 / (1 - q)):
        // chunks whose staged coordinates are coarse relative to the SC's smallest h (far
        // candidates of a tiny-h cluster; error of an in-range pair <= 2^-24 E_i +
        // 2^-23 (E_i + r + X_J), X_J = the staged clusters' max offset, frame.cu) take the
        // fp64 path for every slot
        hmin = warp_fmin(hmin);
        const double ec_i = 5.9604644775390625e-08 * double(Ei) + 1.1920928955078125e-07 * (double(Ei) + double(er));
        // with the global max offset X the whole SC is fine: no per-chunk check
        const bool check_chunks =
            K == SFCNL_KERNEL_DENSITY && 1.7320508075688772 * (ec_i + 1.1920928955078125e-07 * double(X)) > kPiDensityDq * double(hmin);
        __syncwarp();

        bool coincident = false;
        float Ej_run = -1.f;  // running bound of the staged |coordinates| for the guard bands
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
            for (uint32_t h0 = 0; h0 < len; h0 += 32) {
                const uint32_t n = tmin<uint32_t>(32, len - h0);
                const bool have = lane < n;
                const uint32_t my_idx = have ? S.idx[h0 + lane] : 0u;
                const uint32_t my_msk = have ? uint32_t(rec[bb + h0 + lane]) : 0u;
                const int jl0_me = int(my_idx) * CJ - int(p0);
                const bool self_me = have && jl0_me > -CJ && jl0_me < kSC;
                bool coarse = false;
                if (K == SFCNL_KERNEL_DENSITY && check_chunks && !unsafe) {
                    const float xc = warp_fmax(have ? __uint_as_float(A.frame_xcl[my_idx]) : 0.f);
                    coarse = 1.7320508075688772 * (ec_i + 1.1920928955078125e-07 * double(xc)) > kPiDensityDq * double(hmin);
                }

                if (unsafe || coarse) {
                    // every slot through the reference predicate + fp64 kernel
                    for (uint32_t b = 0; b < nicl; ++b) {
                        unsigned mine = __ballot_sync(0xffffffffu, (my_msk >> b) & 1u);
                        const uint32_t il = lane >> 2, jq = lane & 3;
                        const int li = int(b * 8 + il);
                        const double r = S.ir[li];
                        uint32_t c = 0;
                        while (mine) {
                            const uint32_t e = __ffs(mine) - 1;
                            mine &= mine - 1;
                            const uint64_t jb = uint64_t(__shfl_sync(0xffffffffu, my_idx, e)) * CJ;
                            if (r < 0.0) continue;
#pragma unroll
                            for (int s = 0; s < 2; ++s) {
                                const uint64_t j = jb + jq + 4 * s;
                                if ((s == 0 || CJ == 8) && j < A.n) {
                                    const int rc = rare_slot<K>(A, p0 + li, j, dmul(r, r), &S.acc[li][0]);
                                    c += rc > 0, coincident |= rc < 0;
                                }
                            }
                        }
                        if (c) atomicAdd(&S.cnt[li], c);
                    }
                    __syncwarp();
                    continue;
                }

                // ---- stage the chunk's j particles, pair-packed [p][e]
                float Ej = 0.f, Xo = 0.f;
                if (!LJ) {
                    // cluster frame: shift = fl32(minimage(c_J - o)) per entry, s = shift + off
                    float shx = 0.f, shy = 0.f, shz = 0.f;
                    if (have) {
                        const uint64_t c0 = uint64_t(my_idx) * CJ;
                        shx = float(rel(A.x[c0], ox, 0)), shy = float(rel(A.y[c0], oy, 1)), shz = float(rel(A.z[c0], oz, 2));
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t e = uint32_t(u) * 4 + (lane >> 3), jj = lane & 7;
                        const uint32_t ie = __shfl_sync(0xffffffffu, my_idx, e);
                        const float sx = __shfl_sync(0xffffffffu, shx, e), sy = __shfl_sync(0xffffffffu, shy, e);
                        const float sz = __shfl_sync(0xffffffffu, shz, e);
                        if (e >= n) continue;
                        const uint64_t j = uint64_t(ie) * CJ + jj;
                        float vx = kFar, vy = kFar, vz = kFar, vm = 0.f;
                        if (jj < uint32_t(CJ) && j < A.n) {
                            const float4 f = __ldg(A.frame + j);
                            vx = sx + f.x, vy = sy + f.y, vz = sz + f.z, vm = f.w;
                            Ej = fmaxf(Ej, fmaxf(fabsf(vx), fmaxf(fabsf(vy), fabsf(vz))));
                        }
                        float* pa = reinterpret_cast<float*>(&S.sa[jj >> 1][e]) + (jj & 1);
                        float* pb = reinterpret_cast<float*>(&S.sb[jj >> 1][e]) + (jj & 1);
                        pa[0] = vx, pa[2] = vy, pb[0] = vz, pb[2] = vm;
                    }
                    Xo = X;
                } else {
#pragma unroll
                    for (int u0 = 0; u0 < 8; u0 += 4) {
                        double vx[4], vy[4], vz[4];
                        bool val[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t e = uint32_t(u0 + u) * 4 + (lane >> 3), jj = lane & 7;
                            const uint32_t ie = __shfl_sync(0xffffffffu, my_idx, e);
                            const uint64_t j = uint64_t(ie) * CJ + jj;
                            val[u] = e < n && jj < uint32_t(CJ) && j < A.n;
                            vx[u] = vy[u] = vz[u] = 0.0;
                            if (val[u]) vx[u] = A.x[j], vy[u] = A.y[j], vz[u] = A.z[j];
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t e = uint32_t(u0 + u) * 4 + (lane >> 3), jj = lane & 7;
                            if (e >= n) continue;
                            float fx = kFar, fy = kFar, fz = kFar, lx = 0.f, ly = 0.f, lz = 0.f;
                            if (val[u]) {
                                const double qx = rel(vx[u], ox, 0), qy = rel(vy[u], oy, 1), qz = rel(vz[u], oz, 2);
                                fx = float(qx), fy = float(qy), fz = float(qz);
                                lx = float(qx - double(fx)), ly = float(qy - double(fy)), lz = float(qz - double(fz));
                                Ej = fmaxf(Ej, fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))));
                            }
                            float* pa = reinterpret_cast<float*>(&S.sa[jj >> 1][e]) + (jj & 1);
                            float* pb = reinterpret_cast<float*>(&S.sb[jj >> 1][e]) + (jj & 1);
                            float* pc = reinterpret_cast<float*>(&S.sc[jj >> 1][e]) + (jj & 1);
                            pa[0] = fx, pa[2] = fy, pb[0] = fz, pb[2] = lx, pc[0] = ly, pc[2] = lz;
                        }
                    }
                }
                Ej = warp_fmax(Ej);
                // per-i thresholds: coordinate errors <= 2^-24 Ei (i side) and
                // 2^-24 Ej (fp64 staging) or 2^-23 (Ej + X) (cluster frame)
                // (the band only widens with Ej: recomputed when a chunk raises the running bound)
                const bool redo = Ej > Ej_run;
                if (redo) Ej_run = fmaxf(Ej, Ej_run * 1.0625f);
                const double ecoord = 5.9604644775390625e-08 * double(Ei) +
                                      (LJ ? 5.9604644775390625e-08 * double(Ej_run) : 1.1920928955078125e-07 * (double(Ej_run) + double(Xo)));
#pragma unroll
                for (int s = 0; s < 2 && redo; ++s) {
                    const uint32_t k = lane + 32u * s;
                    const uint32_t slot = (k & 7) * 8 + (k >> 3);
                    const double r = S.ir[k];
                    float lo = -1.f, hi = -1.f;
                    if (r >= 0.0) {
                        const double r2 = dmul(r, r);
                        const double ex = ecoord + 5.9604644775390625e-08 * r;
                        const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
                        lo = __double2float_rd(r2 - guard);
                        hi = __double2float_ru(r2 + guard);
                    }
                    S.ib[slot].x = lo, S.ib[slot].y = hi;
                }

                // ---- items (b << 5 | e), b-major; non-self entries first
                uint32_t nItems = 0;
#pragma unroll 1
                for (int pass = 0; pass < 2; ++pass) {
                    for (uint32_t b = 0; b < nicl; ++b) {
                        const bool in = ((my_msk >> b) & 1u) && (self_me == (pass == 1));
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        if (in) S.items[nItems + __popc(bal & ltmask)] = uint8_t((b << 5) | lane);
                        nItems += __popc(bal);
                    }
                }
                __syncwarp();

                // ---- rounds: one item per lane
                for (uint32_t t0 = 0; t0 < nItems; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    const bool valid = t < nItems;
                    const uint32_t it8 = valid ? S.items[t] : 0u;
                    const uint32_t e = it8 & 31u, b = it8 >> 5;
                    const int jl0 = __shfl_sync(0xffffffffu, jl0_me, e);
                    const int self_e = __shfl_sync(0xffffffffu, self_me ? 1 : 0, e);
                    const bool self = valid && self_e;
                    ulonglong2 Ja[4], Jb[4], Jc[LJ ? 4 : 1];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        Ja[p] = reinterpret_cast<const ulonglong2&>(S.sa[p][e]);
                        Jb[p] = reinterpret_cast<const ulonglong2&>(S.sb[p][e]);
                        if (LJ) Jc[p] = reinterpret_cast<const ulonglong2&>(S.sc[p][e]);
                    }
                    uint32_t band_rows = 0;
                    unsigned long long close_bits = 0;  // LJ: in-range slots closer than kLjClose * sigma
                    // one row = i (b, ii) against the entry's 8 j slots; SELF rows drop i == j
                    auto rows = [&](auto SELF) {
                        constexpr bool kSelf = decltype(SELF)::value;
#pragma unroll 1
                        for (int ii = 0; ii < 8; ++ii) {
                            const float4 I = S.ia[ii * 8 + b];
                            const float4 T = S.ib[ii * 8 + b];
                            const float lo = valid ? T.x : -1.f, hi = valid ? T.y : -1.f;
                            const f2 xi2 = f2p(I.x, I.x), yi2 = f2p(I.y, I.y), zi2 = f2p(I.z, I.z);
                            f2 lxi2 = 0, lyi2 = 0, lzi2 = 0;
                            if (LJ) {
                                const float lzi = S.ic[ii * 8 + b];
                                lxi2 = f2p(T.z, T.z), lyi2 = f2p(T.w, T.w), lzi2 = f2p(lzi, lzi);
                            }
                            f2 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, nin = 0, nhi = 0;
                            uint32_t crow = 0;
                            const int iself = kSelf && self ? int(b * 8 + ii) - jl0 : -1;
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                f2 dx = f2sub(xi2, f2lo(Ja[p]));
                                f2 dy = f2sub(yi2, f2hi(Ja[p]));
                                f2 dz = f2sub(zi2, f2lo(Jb[p]));
                                if (LJ) {
                                    dx = f2add(dx, f2sub(lxi2, f2hi(Jb[p])));
                                    dy = f2add(dy, f2sub(lyi2, f2lo(Jc[p])));
                                    dz = f2add(dz, f2sub(lzi2, f2hi(Jc[p])));
                                }
                                float d2a, d2b;
                                f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                                if (kSelf) {
                                    if (iself == 2 * p) d2a = kFar;
                                    if (iself == 2 * p + 1) d2b = kFar;
                                }
                                const float ma = fset_lt(d2a, lo), mb = fset_lt(d2b, lo);
                                nin = f2add(nin, f2p(ma, mb));
                                nhi = f2add(nhi, f2p(fset_le(d2a, hi), fset_le(d2b, hi)));
                                if (K == SFCNL_KERNEL_DENSITY) {
                                    // W(q)/(2 sigma) = max(1-q,0)^3 - 4 max(1/2-q,0)^3
                                    // max(1 - q, 0) and max(1/2 - q, 0) as saturated scalar fmas
                                    // (q = |d| / h >= 0, so the clamp at 1 never binds): four
                                    // FFMA.SAT instead of FMUL2 + FFMA2 + FADD2 + four FMNMX
                                    const float sa = sqrt_ftz(d2a), sb = sqrt_ftz(d2b);
                                    const f2 tt = f2p(__saturatef(fmaf(-sa, I.w, 1.f)), __saturatef(fmaf(-sb, I.w, 1.f)));
                                    const f2 uu = f2p(__saturatef(fmaf(-sa, I.w, 0.5f)), __saturatef(fmaf(-sb, I.w, 0.5f)));
                                    const f2 t3 = f2mul(f2mul(tt, tt), tt), u3 = f2mul(f2mul(uu, uu), uu);
                                    const f2 wv = f2fma(f2p(-4.f, -4.f), u3, t3);
                                    acc0 = f2fma(NM ? f2hi(Jb[p]) : f2mul(f2hi(Jb[p]), f2p(ma, mb)), wv, acc0);
                                } else if (LJ) {
                                    // close pairs leave the fp32 sums (evaluated in fp64 below)
                                    const bool cla = ma != 0.f && d2a < close2, clb = mb != 0.f && d2b < close2;
                                    crow |= (cla ? 1u : 0u) << (2 * p);
                                    crow |= (clb ? 1u : 0u) << (2 * p + 1);
                                    const f2 inv2 = f2p(ma != 0.f && !cla ? rcp_ftz(d2a) : 0.f, mb != 0.f && !clb ? rcp_ftz(d2b) : 0.f);
                                    // 24 eps and 4 eps are applied to the row sums (LjKernel, builtin_kernels.hpp:41-77)
                                    const f2 s2 = f2mul(f2p(sig2, sig2), inv2);
                                    const f2 s6 = f2mul(f2mul(s2, s2), s2);
                                    f2 cf = f2mul(inv2, f2mul(s6, f2fma(f2p(2.f, 2.f), s6, f2p(-1.f, -1.f))));
                                    f2 ee = f2fma(s6, s6, f2mul(s6, f2p(-1.f, -1.f)));
                                    if (K == SFCNL_KERNEL_LJ_COULOMB) {  // eps may be 0: no folding
                                        cf = f2mul(cf, f2p(eps24, eps24));
                                        ee = f2mul(ee, f2p(eps4, eps4));
                                    }
                                    if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                        const uint64_t i = p0 + b * 8 + ii;
                                        const uint64_t jb = uint64_t(S.idx[h0 + e]) * CJ + 2 * p;
                                        const float qi = float(A.ck * A.q[i]);
                                        const float qa = ma != 0.f && !cla ? qi * float(A.q[jb]) : 0.f;
                                        const float qb = mb != 0.f && !clb && jb + 1 < A.n ? qi * float(A.q[jb + 1]) : 0.f;
                                        float ra, rb;
                                        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(d2a));
                                        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(d2b));
                                        const f2 qr = f2mul(f2p(qa, qb), f2p(ra, rb));
                                        ee = f2add(ee, qr);
                                        cf = f2fma(qr, inv2, cf);
                                    }
                                    acc0 = f2fma(cf, dx, acc0);
                                    acc1 = f2fma(cf, dy, acc1);
                                    acc2 = f2fma(cf, dz, acc2);
                                    acc3 = f2add(acc3, ee);
                                }
                            }
                            float ni0, ni1, nh0, nh1;
                            f2u(nin, ni0, ni1);
                            f2u(nhi, nh0, nh1);
                            const float ncnt = ni0 + ni1;
                            if (ncnt != nh0 + nh1) band_rows |= 1u << ii;  // a slot with d2 in [lo, hi]
                            if (LJ) close_bits |= (unsigned long long)crow << (8 * ii);
                            float* pp = &S.part[ii][0][lane];
                            pp[NO * (32 + SFCNL_PI_PAD)] = ncnt;
                            if (K != SFCNL_KERNEL_COUNT) {
                                const f2 accs[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
                                for (int o = 0; o < NO; ++o) {
                                    float a0, a1;
                                    f2u(accs[o], a0, a1);
                                    pp[o * (32 + SFCNL_PI_PAD)] = K == SFCNL_KERNEL_LJ ? (a0 + a1) * (o < 3 ? eps24 : eps4) : a0 + a1;
                                }
                            }
                        }
                    };
                    if (__any_sync(0xffffffffu, self)) rows(BoolC<true>());
                    else rows(BoolC<false>());
                    // LJ close pairs: fp64 from the staged hi/lo coordinates (exact SC-frame
                    // values); the coincidence range goes to the reference path
                    if (LJ && valid && close_bits) {
                        const uint64_t jb0 = uint64_t(S.idx[h0 + e]) * CJ;
                        while (close_bits) {
                            const int k = __ffsll(close_bits) - 1;
                            close_bits &= close_bits - 1;
                            const int ii = k >> 3, jj = k & 7;
                            const int li = int(b * 8 + ii);
                            const float4 I = S.ia[ii * 8 + b];
                            const float4 T = S.ib[ii * 8 + b];
                            const float lzi = S.ic[ii * 8 + b];
                            const float* pa = reinterpret_cast<const float*>(&S.sa[jj >> 1][e]) + (jj & 1);
                            const float* pb = reinterpret_cast<const float*>(&S.sb[jj >> 1][e]) + (jj & 1);
                            const float* pc = reinterpret_cast<const float*>(&S.sc[jj >> 1][e]) + (jj & 1);
                            const double ddx = (double(I.x) - double(pa[0])) + (double(T.z) - double(pb[2]));
                            const double ddy = (double(I.y) - double(pa[2])) + (double(T.w) - double(pc[0]));
                            const double ddz = (double(I.z) - double(pb[0])) + (double(lzi) - double(pc[2]));
                            const double dd2 = ddx * ddx + ddy * ddy + ddz * ddz;
                            float* pp = &S.part[ii][0][lane];
                            if (!(dd2 >= double(kLjTiny2) * sig2d)) {
                                // coincidence range: the reference predicate + fp64 kernel
                                pp[NO * (32 + SFCNL_PI_PAD)] -= 1.f;
                                const int rc = rare_slot<K>(A, p0 + li, jb0 + jj, dmul(S.ir[li], S.ir[li]), &S.acc[li][0]);
                                if (rc > 0) atomicAdd(&S.cnt[li], 1u);
                                coincident |= rc < 0;
                                continue;
                            }
                            const double in2 = 1.0 / dd2;
                            const double s2d = sig2d * in2, s6d = s2d * s2d * s2d;
                            double coef = eps24d * in2 * s6d * (2.0 * s6d - 1.0);
                            double en = eps4d * s6d * (s6d - 1.0);
                            if (K == SFCNL_KERNEL_LJ_COULOMB) {
                                const double qq = A.ck * A.q[p0 + li] * A.q[jb0 + jj], irr = sqrt(in2);
                                en += qq * irr;
                                coef += qq * irr * in2;
                            }
                            constexpr int R = 32 + SFCNL_PI_PAD;
                            pp[0] += float(coef * ddx), pp[R] += float(coef * ddy);
                            pp[2 * R] += float(coef * ddz), pp[3 * R] += float(en);
                        }
                    }
                    // band rows: the reference's predicate decides the slots in [lo, hi]
                    if (valid && band_rows) {
                        for (int ii = 0; ii < 8; ++ii) {
                            if (!((band_rows >> ii) & 1u)) continue;
                            const int li = int(b * 8 + ii);
                            const float4 I = S.ia[ii * 8 + b];
                            const float4 T = S.ib[ii * 8 + b];
                            const float lzi = LJ ? S.ic[ii * 8 + b] : 0.f;
                            const double r = S.ir[li];
                            for (int jj = 0; jj < 8; ++jj) {
                                if (self && int(b * 8 + ii) - jl0 == jj) continue;
                                const float* pa = reinterpret_cast<const float*>(&S.sa[jj >> 1][e]) + (jj & 1);
                                const float* pb = reinterpret_cast<const float*>(&S.sb[jj >> 1][e]) + (jj & 1);
                                const float* pc = reinterpret_cast<const float*>(&S.sc[jj >> 1][e]) + (jj & 1);
                                float dx = I.x - pa[0], dy = I.y - pa[2], dz = I.z - pb[0];
                                if (LJ) dx = dx + (T.z - pb[2]), dy = dy + (T.w - pc[0]), dz = dz + (lzi - pc[2]);
                                const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                                if (d2 < T.x || d2 > T.y) continue;
                                const uint64_t j = uint64_t(S.idx[h0 + e]) * CJ + jj;
                                if (jj >= CJ || j >= A.n) continue;
                                const int rc = rare_slot<K>(A, p0 + li, j, dmul(r, r), &S.acc[li][0]);
                                if (rc > 0) atomicAdd(&S.cnt[li], 1u);
                                coincident |= rc < 0;
                            }
                        }
                    }
                    __syncwarp();
                    // deterministic reduction of the round's partial sums per i (item order)
                    {
                        unsigned mb_[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) mb_[q] = __ballot_sync(0xffffffffu, valid && b == uint32_t(q));
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const uint32_t i = lane + 32u * s;
                            const uint32_t ib_ = i >> 3, ii = i & 7;
                            unsigned m = 0;
#pragma unroll
                            for (int q = 0; q < 8; ++q) m = (ib_ == uint32_t(q)) ? mb_[q] : m;
                            if (!m) continue;
                            float sum[NO + 1];
#pragma unroll
                            for (int o = 0; o <= NO; ++o) sum[o] = 0.f;
                            while (m) {
                                const uint32_t tl = __ffs(m) - 1;
                                m &= m - 1;
#pragma unroll
                                for (int o = 0; o <= NO; ++o) sum[o] += S.part[ii][o][tl];
                            }
                            S.cnt[i] += uint32_t(sum[NO]);
                            if (K == SFCNL_KERNEL_DENSITY) {
                                S.acc[i][0] += S.iscale[i] * double(sum[0]);
                            } else if (LJ) {
#pragma unroll
                                for (int o = 0; o < NO; ++o) S.acc[i][o] += double(sum[o]);
                            }
                        }
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
                        for (int o = 0; o < NO; ++o) A.out[o][i] = S.acc[k][o];
                    }
                    A.cnt[i] = S.cnt[k];
                }
            }
        }
        __syncwarp();  // the warp's slice is reused by its next SC
    }
}
