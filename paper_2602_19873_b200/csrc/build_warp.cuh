// Warp-per-super-cluster list build for gather stores with ci == 8, cj in {4, 8}
// (included by build.cu after build_fast.cuh, inside namespace sfcnl_cu::{anon}).
//
// Same results as build_sc (and so as build_neighbor_store, neighbor_build.cpp:74-184),
// restructured for the GPU: every warp takes the next super-cluster (SC) from a
// global counter and builds it alone, so there are no block barriers; the warps of
// an SM hide each other's memory latency.
//
//  1. geometry: SC box = sequential union of its i-cluster boxes (every lane,
//     neighbor_build.cpp:113-118); i particles relative to the SC's first particle
//     (fp64, per-particle minimum image) rounded to fp32, i-cluster fp32 boxes.
//  2. traversal (collect_candidates, :43-65): level-synchronous BFS over the octree
//     with an ORDERED frontier in the warp's shared memory; 32 nodes tested per
//     step (exact fp64 aabb_dist_sq), warp scans place children / tagged accepted
//     leaves, so the accepted leaves come out in key order.
//  3. candidates: per accepted leaf its j-cluster range minus the cluster shared with
//     the previous leaf (`out.back() != j`, :57-58); a prefix sum over leaves lets each
//     lane locate its candidate of a 32-wide chunk by binary search.
//  4. masks (:128-161) per chunk of 32 candidates: stage the j particles in fp32 in
//     the SC frame from the cluster-frame copy (frame.cu), conservative fp32 AABB
//     prefilter (lane = candidate), then ONE (i-cluster, candidate) ITEM PER LANE: the
//     lane holds the candidate's 8 j particles in registers and walks the 8 i rows
//     (two slots per FFMA2), tracking the row minimum of d2; a hit is d2 < lo (exact
//     d2 < r_i^2), a row minimum in [lo, hi] is decided by the reference's fp64 pair
//     predicate and prefilter (see build_fast.cuh for the argument).
//     SCs whose periodic images are ambiguous in the SC frame run the reference
//     loop in fp64 (lane = candidate).
//  5. entries with mask != 0 are compacted in order (ballot), then encoded by the
//     warp (codec::encode, nibble_codec.cpp:56-134) into a byte buffer that aliases
//     the staging area, bump-allocated into the scratch and copied out.
// An SC that exceeds a capacity (frontier, entries, bytes) is listed for the
// global-memory fallback kernel (k_build_global), which runs the generic build_sc.
constexpr int kBwWarps = 4;
#define SFCNL_UNLIKELY(c) __builtin_expect(!!(c), 0)  // cold blocks placed out of the hot path
// main tier: no SC of the C2 / C3 workloads exceeds these (the medium tier takes the rest)
constexpr uint32_t kBwF = 320;   // frontier entries per buffer
constexpr uint32_t kBwE = 384;   // entries per SC (~170 at 200 neighbours)
constexpr uint32_t kBwBytes = 2560;  // encoded bytes (aliases the frontier)
constexpr uint32_t kLeafCacheCap = 256;
#ifndef SFCNL_BW_SZ8
#define SFCNL_BW_SZ8 0
#endif
constexpr bool kBwSz8 = SFCNL_BW_SZ8;  // accepted leaves kept per SC by halo marking

// Per-warp shared-memory slice. Two capacity tiers: the main kernel runs every SC with
// the small one (5 CTAs x 4 warps per SM); SCs that exceed it (dense lists, wide skins,
// 8x4 clusters at high neighbour counts) are re-run from the overflow list with the
// medium one (3 CTAs x 4 warps per SM); only SCs beyond that go to k_build_global.
// symmetric mode: per-j guard-band thresholds of the staged chunk ([p][candidate] pairs)
template <bool SYM>
struct BwSymJ {
    float2 slo[4][32], shi[4][32];
};
template <>
struct BwSymJ<false> {};

template <uint32_t F, uint32_t E, uint32_t B, bool SYM = false, bool BFS = true>
struct BwSmemT {
    static constexpr uint32_t kF = F, kE = E, kB = B;
    static constexpr bool kSym = SYM;
    static constexpr bool kBfs = BFS;  // false: leaves from the traversal kernel's cache only
    union {
        struct {
            uint32_t fa[F], fb[F];  // traversal frontier, then per-leaf candidate prefix
        } t;
        uint8_t ebuf[B];  // encoder output (after the masks: the frontier is dead)
    } u;
    float4 sa[4][32];  // staged j pairs [p][candidate]: {x_2p, x_2p+1, y_2p, y_2p+1}
    // {z_2p, z_2p+1 (, -, -)}: 16-byte rows measured faster in the traversing kernel
    std::conditional_t<BFS && !kBwSz8, float4, float2> sz[4][32];
    float4 ia[64];     // [ii*8 + b] {x, y, z, lo} SC frame + cutoff threshold (guard band below)
    float ihi[64];     // [ii*8 + b] hi threshold (guard band above)
    float iab[8][6];
    float pthr[8];
    uint32_t cmask[32];
    uint8_t items[256];
    uint32_t eidx[E];
    uint8_t emsk[E];
    BwSymJ<SYM> sy;
};
using BwSmem = BwSmemT<kBwF, kBwE, kBwBytes>;
// gather main tier after the traversal kernel (k_halo_warp fills the leaf cache, <= 256
// leaves per SC): no traversal code, SCs without cached leaves go to the medium tier
using BwSmemCached = BwSmemT<kLeafCacheCap, kBwE, 2048, false, false>;
using BwSmemM = BwSmemT<1024, 1024, 8192>;
using BwSmemSym = BwSmemT<kBwF, kBwE, kBwBytes, true>;
using BwSmemMSym = BwSmemT<1024, 1024, 8192, true>;

// Guard band on a squared distance near r^2 when every coordinate difference carries
// an absolute error <= ecoord + 2^-24 r (see pass.cu); factor 4 margin.
__device__ __forceinline__ double guard_band(double r, double r2, double ecoord) {
    const double ex = ecoord + 5.9604644775390625e-08 * r;
    return 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Ordered-frontier BFS of one SC over the octree (collect_candidates,
// neighbor_build.cpp:43-65) by one warp: 32 nodes per step, exact fp64 aabb_dist_sq;
// warp scans place children and tagged accepted leaves, so the accepted leaves end
// up in key order in *out (one of the two buffers). Returns their number, or ~0u
// when the frontier exceeds kBwF.
//
// Gather traversal pre-test (A.ngeo32): the box gap in fp32 from boxes rounded to
// nearest. Every input carries an error <= u M (u = 2^-24, M >= any |bound| incl. the
// periodic shifts), the shift and the difference one rounding each, so a gap is off by
// at most d = u (5 M + r) near the cutoff, and the squared distance by
// B = 2 sqrt(3) r d + 3 d^2 + 3 u r^2; d2_f32 > r^2 + 2B rejects, d2_f32 < r^2 - 2B
// accepts (d2 - err(d2) grows with d2), anything between runs the exact fp64 test.
__device__ __forceinline__ float gap32(float alo, float ahi, float blo, float bhi) {
    return fmaxf(fmaxf(alo, blo) - fminf(ahi, bhi), 0.f);
}

__device__ __forceinline__ uint32_t warp_bfs(const BuildArgs& A, const Geo& scg, double r2, uint32_t* fa,
                                             uint32_t* fb, uint32_t** out, uint32_t cap = kBwF) {
    const unsigned lane = lane_id();
    const bool pre = A.ngeo32 != nullptr;
    float slo[3], shi[3], L32[3], r2lo = 0.f, r2hi = 0.f;
    if (pre) {
#pragma unroll
        for (int d = 0; d < 3; ++d) slo[d] = float(scg.lo[d]), shi[d] = float(scg.hi[d]), L32[d] = float(A.box.len[d]);
        const double u = 5.9604644775390625e-08, r = sqrt(r2);
        const double dl = u * (5.0 * double(A.trav_m) + r);
        const double B = 2.0 * (3.4641016151377544 * r * dl + 3.0 * dl * dl + 3.0 * u * r2) + 1e-12 * r2 + 1e-300;
        r2lo = __double2float_rd(r2 - B), r2hi = __double2float_ru(r2 + B);
    }
    if (lane == 0) fa[0] = 0;
    uint32_t nA = 1;
    __syncwarp();
    for (;;) {
        uint32_t nB = 0;
        bool expanded = false;
        for (uint32_t base = 0; base < nA; base += 32) {
            const uint32_t k = base + lane;
            uint32_t emit = 0, e = 0;
            int32_t fc = -1;
            if (k < nA) {
                e = fa[k];
                if (e & kTag) {
                    emit = 1;
                } else {
                    const Node nd = A.nodes[e];
                    if (nd.pend > nd.pbegin) {
                        int acc = -1;  // pre-test: 1 accept, 0 reject, -1 undecided
                        if (pre) {
                            const float4 lo = A.ngeo32[2 * e], hi = A.ngeo32[2 * e + 1];
                            const float bl[3] = {lo.x, lo.y, lo.z}, bh[3] = {hi.x, hi.y, hi.z};
                            float d2f = 0.f;
#pragma unroll
                            for (int d = 0; d < 3; ++d) {
                                float g = gap32(slo[d], shi[d], bl[d], bh[d]);
                                if (A.box.per[d]) {
                                    g = fminf(g, gap32(slo[d], shi[d], bl[d] - L32[d], bh[d] - L32[d]));
                                    g = fminf(g, gap32(slo[d], shi[d], bl[d] + L32[d], bh[d] + L32[d]));
                                }
                                d2f = fmaf(g, g, d2f);
                            }
                            acc = d2f > r2hi ? 0 : (d2f < r2lo ? 1 : -1);
                        }
                        if (acc < 0) {
                            const Geo ng = A.ngeo[e];
                            double rr2 = r2;
                            if (A.symmetric) {  // scale * max(sc_maxh, node_maxh) (neighbor_build.cpp:122-125)
                                const double rr = dmul(A.scale, smax(scg.maxh, ng.maxh));
                                rr2 = dmul(rr, rr);
                            }
                            acc = !(aabb_dist_sq(scg, ng, A.box) > rr2);
                        }
                        if (acc) {
                            fc = nd.first_child;
                            emit = fc < 0 ? 1 : 8;
                        }
                    }
                }
            }
            const uint32_t inc = warp_incl_scan(emit);
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            if (nB + tot > cap) return ~0u;
            const uint32_t at = nB + inc - emit;
            if (emit == 1) fb[at] = e | kTag;
            if (emit == 8) {
#pragma unroll
                for (int c = 0; c < 8; ++c) fb[at + c] = uint32_t(fc + c);
            }
            expanded |= __any_sync(0xffffffffu, emit == 8);
            nB += tot;
        }
        __syncwarp();
        uint32_t* t = fa;
        fa = fb, fb = t;
        nA = nB;
        if (!expanded) break;
    }
    *out = fa;
    return nA;
}

// SC box = sequential union of its i-cluster boxes (neighbor_build.cpp:113-118) and the
// traversal radius; every lane.
__device__ __forceinline__ void sc_box(const BuildArgs& A, uint64_t icl_base, uint32_t nicl, Geo& scg, double& r2) {
    geo_init(scg);
    for (uint32_t b = 0; b < nicl; ++b) {
        const Geo g = A.igeo[icl_base + b];
        geo_extend(scg, g);
        scg.maxh = smax(scg.maxh, g.maxh);
    }
    const double r = dmul(A.scale, scg.maxh);
    r2 = dmul(r, r);
}

// unsafe SCs: the reference's mask loop in fp64 for one candidate (lane = candidate,
// neighbor_build.cpp:128-161)
template <bool SYM>
__device__ __forceinline__ uint32_t unsafe_mask(const BuildArgs& A, uint32_t cand, uint64_t icl_base, uint32_t nicl) {
    const uint32_t cj = A.cj;
    uint32_t mask = 0;
    const Geo jg = A.jgeo[cand];
    const uint64_t jb = uint64_t(cand) * cj, je = tmin<uint64_t>(jb + cj, A.n);
    for (uint32_t b = 0; b < nicl; ++b) {
        if (SYM && (icl_base + b) * 8 > jb) continue;  // half-list rule (neighbor_build.cpp:133)
        const Geo ig = A.igeo[icl_base + b];
        const double pre_r = dmul(A.scale, SYM ? smax(ig.maxh, jg.maxh) : ig.maxh);
        if (aabb_dist_sq(ig, jg, A.box) > dmul(pre_r, pre_r)) continue;
        const uint64_t ib = (icl_base + b) * 8, ie = tmin<uint64_t>(ib + 8, A.n);
        bool hit = false;
        for (uint64_t i = ib; i < ie && !hit; ++i) {
            const double xi = A.x[i], yi = A.y[i], zi = A.z[i];
            const double rr = dmul(A.scale, A.h[i]);
            for (uint64_t j = jb; j < je; ++j) {
                if (i == j) continue;
                const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, nullptr, nullptr, nullptr);
                const double rs = SYM ? dmul(A.scale, smax(A.h[i], A.h[j])) : rr;
                if (d2 <= dmul(rs, rs)) {
                    hit = true;
                    break;
                }
            }
        }
        if (hit) mask |= 1u << b;
    }
    return mask;
}

// an item whose fp32 row minima fell inside the guard band: the reference's exact pair
// predicate on those rows, then its prefilter (neighbor_build.cpp:136-155) -- any
// exact hit suffices
template <bool SYM>
__device__ __forceinline__ bool band_item(const BuildArgs& A, uint64_t p0, uint64_t icl_base, uint32_t b, uint32_t cc,
                                       uint32_t band_rows) {
#ifdef SFCNL_PHASE_PROF
    atomicAdd(A.prof + 10, 1ull);
#endif
    const uint32_t cj = A.cj;
    const uint64_t jb = uint64_t(cc) * cj;
    bool ex = false;
    for (int ii = 0; ii < 8 && !ex; ++ii) {
        if (!((band_rows >> ii) & 1u)) continue;
        const uint64_t gi = p0 + b * 8 + ii;
        for (uint32_t jj = 0; jj < cj && !ex; ++jj) {
            if (jb + jj >= A.n || jb + jj == gi) continue;
            ex = exact_hit(A, A.x[gi], A.y[gi], A.z[gi], A.h[gi], jb + jj);
        }
    }
    if (!ex) return false;
    const Geo ig = A.igeo[icl_base + b];
    const double pr = dmul(A.scale, SYM ? smax(ig.maxh, A.jgeo[cc].maxh) : ig.maxh);
    return !(aabb_dist_sq(ig, A.jgeo[cc], A.box) > dmul(pr, pr));
}

// Returns false when a capacity is exceeded (nothing published).
#ifdef SFCNL_PHASE_PROF
#define PHASE(k)                                                                   \
    do {                                                                           \
        const long long _t = clock64();                                            \
        if (lane == 0) atomicAdd(A.prof + (k), (unsigned long long)(_t - _tprev)); \
        _tprev = _t;                                                               \
    } while (0)
#else
#define PHASE(k) \
    do {         \
    } while (0)
#endif

template <class Sm>
__device__ bool build_sc_warp(const BuildArgs& A, Sm& S, uint64_t sc) {
    constexpr bool SYM = Sm::kSym;
    const unsigned lane = lane_id();
#ifdef SFCNL_PHASE_PROF
    long long _tprev = clock64();
#endif
    const uint64_t icl_base = sc * 8;
    const uint32_t nicl = uint32_t(tmin<uint64_t>(icl_base + 8, A.num_icl) - icl_base);
    const uint64_t p0 = sc * kSC;
    const uint32_t np = uint32_t(tmin<uint64_t>(p0 + kSC, A.n) - p0);
    const uint32_t cj = A.cj;

    // ---- 1. SC geometry (sequential union, as sc_geometry) and the i side
    Geo scg;
    double r2;
    sc_box(A, icl_base, nicl, scg, r2);
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
    double ri[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t k = lane + 32u * s;
        float fx = 1e30f, fy = 1e30f, fz = 1e30f;
        ri[s] = -1.0;
        if (k < np) {
            const double qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
            fx = float(qx), fy = float(qy), fz = float(qz);
            eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
            ri[s] = dmul(A.scale, A.h[p0 + k]);
            er = fmaxf(er, float(ri[s]));
        }
        S.ia[(k & 7) * 8 + (k >> 3)] = make_float4(fx, fy, fz, 0.f);
    }
    eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
    // per-particle (i) and per-cluster (j, cluster frame) images against the SC origin are
    // exact for every in-range pair when max|rel_i| + max r + X < 0.49 L (frame.cu)
    const float Xx = __uint_as_float(A.frame_x[0]), Xy = __uint_as_float(A.frame_x[1]), Xz = __uint_as_float(A.frame_x[2]);
    const bool unsafe = (A.box.per[0] && double(eax) + double(er) + double(Xx) >= 0.49 * A.box.len[0]) ||
                        (A.box.per[1] && double(eay) + double(er) + double(Xy) >= 0.49 * A.box.len[1]) ||
                        (A.box.per[2] && double(eaz) + double(er) + double(Xz) >= 0.49 * A.box.len[2]);
    const float Xo = fmaxf(Xx, fmaxf(Xy, Xz));
    const float Ei = fmaxf(eax, fmaxf(eay, eaz));
    __syncwarp();
    if (lane < nicl) {  // fp32 boxes of the i-clusters (SC frame)
        float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
        for (uint32_t k = lane * 8; k < tmin<uint32_t>(lane * 8 + 8, np); ++k) {
            const float4 v = S.ia[(k & 7) * 8 + lane];
            lo[0] = fminf(lo[0], v.x), hi[0] = fmaxf(hi[0], v.x);
            lo[1] = fminf(lo[1], v.y), hi[1] = fmaxf(hi[1], v.y);
            lo[2] = fminf(lo[2], v.z), hi[2] = fmaxf(hi[2], v.z);
        }
        for (int d = 0; d < 3; ++d) S.iab[lane][d] = lo[d], S.iab[lane][3 + d] = hi[d];
    }

    PHASE(0);
    // ---- 2. ordered-frontier BFS (exact fp64 node test)
    uint32_t* fa;
    uint32_t nA = ~0u;
    if (!SYM && A.leaf_cache) {  // halo marking of this range already traversed (same BFS, same order)
        const uint32_t cnt = A.leaf_count[sc - A.leaf_sc0];
        if (cnt != ~0u) {
            const uint32_t* src = A.leaf_cache + (sc - A.leaf_sc0) * kLeafCacheCap;
            for (uint32_t k = lane; k < cnt; k += 32) S.u.t.fa[k] = src[k];
            __syncwarp();
            fa = S.u.t.fa, nA = cnt;
        }
    }
    if (nA == ~0u) {
        if constexpr (Sm::kBfs) nA = warp_bfs(A, scg, r2, S.u.t.fa, S.u.t.fb, &fa, Sm::kF);
        else return false;  // not cached: the medium tier traverses
    }
    if (nA == ~0u) return false;
    uint32_t* fb = fa == S.u.t.fa ? S.u.t.fb : S.u.t.fa;

    PHASE(1);
    // ---- 3. candidate ranges per accepted leaf: fa[k] <- first candidate, fb[k] <- prefix
    uint32_t nC = 0;
    {
        uint32_t prev_last = 0xffffffffu;  // last cluster of the previous leaf
        for (uint32_t base = 0; base < nA; base += 32) {
            const uint32_t k = base + lane;
            uint32_t f = 0, l = 0;
            if (k < nA) {
                const Node nd = A.nodes[fa[k] & ~kTag];
                f = nd.pbegin / cj, l = (nd.pend - 1) / cj;
            }
            uint32_t pl = __shfl_up_sync(0xffffffffu, l, 1);
            if (lane == 0) pl = prev_last;
            uint32_t start = f, cnt = 0;
            if (k < nA) {
                if (k > 0 && pl == f) start = f + 1;
                cnt = l + 1 - start;
            }
            const uint32_t inc = warp_incl_scan(cnt);
            __syncwarp();
            if (k < nA) fa[k] = start, fb[k] = nC + inc - cnt;
            nC += __shfl_sync(0xffffffffu, inc, 31);
            prev_last = __shfl_sync(0xffffffffu, l, 31);
        }
        __syncwarp();
    }

    PHASE(2);
    // ---- 4. masks, chunk by chunk; 5a. ordered compaction of mask != 0
    uint32_t nE = 0;
    float Ej_run = -1.f;               // running max of the staged |coordinates| (guard bands)
    double ecoord_cur = 0.0;           // coordinate error bound of the current thresholds
    double pr_me = 0.0, pr2_me = 0.0;  // prefilter radius of i-cluster `lane` (neighbor_build.cpp:136)
    if (lane < nicl) pr_me = dmul(A.scale, A.igeo[icl_base + lane].maxh), pr2_me = dmul(pr_me, pr_me);
    for (uint32_t c0 = 0; c0 < nC; c0 += 32) {
        const uint32_t n = tmin<uint32_t>(32, nC - c0);
        const bool valid = lane < n;
        uint32_t cand = 0;
        if (valid) {  // leaf k = last with prefix <= pos
            const uint32_t pos = c0 + lane;
            uint32_t lo = 0, hi = nA;  // fb[lo] <= pos < fb[hi]
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (fb[mid] <= pos) lo = mid;
                else hi = mid;
            }
            cand = fa[lo] + (pos - fb[lo]);
        }
        const int jl0 = int(cand) * int(cj) - int(p0);
        const unsigned selfm = __ballot_sync(0xffffffffu, valid && jl0 >= -7 && jl0 < kSC);
        uint32_t mask = 0;
        if (SFCNL_UNLIKELY(unsafe)) {
            // reference loop in fp64, lane = candidate (neighbor_build.cpp:128-161)
            if (valid) mask = unsafe_mask<SYM>(A, cand, icl_base, nicl);
        } else {
            // stage (cluster frame, frame.cu): shift = fl32(minimage(c_J - o)) per candidate,
            // s = shift + off per particle; [p][candidate] pair-packed. Every load of the
            // chunk (origins: lane = candidate; offsets: lane = particle) is issued first.
            double cx = 0.0, cy = 0.0, cz = 0.0;
            if (valid) {
                const uint64_t c0 = uint64_t(cand) * cj;
                cx = A.x[c0], cy = A.y[c0], cz = A.z[c0];
            }
            float4 fo[8];
            uint32_t okm = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t e = uint32_t(u) * 4 + (lane >> 3), jj = lane & 7;
                const uint32_t ce = __shfl_sync(0xffffffffu, cand, e);
                const uint64_t j = uint64_t(ce) * cj + jj;
                const bool ok = e < n && jj < cj && j < A.n;
                fo[u] = ok ? __ldg(A.frame + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                okm |= uint32_t(ok) << u;
            }
            float shx = 0.f, shy = 0.f, shz = 0.f;
            if (valid) shx = float(rel(cx, ox, 0)), shy = float(rel(cy, oy, 1)), shz = float(rel(cz, oz, 2));
            float Ej = 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t e = uint32_t(u) * 4 + (lane >> 3), jj = lane & 7;
                const float sx = __shfl_sync(0xffffffffu, shx, e), sy = __shfl_sync(0xffffffffu, shy, e);
                const float sz = __shfl_sync(0xffffffffu, shz, e);
                if (e >= n) continue;
                float vx = 1e30f, vy = 1e30f, vz = 1e30f;
                if ((okm >> u) & 1u) {
                    vx = sx + fo[u].x, vy = sy + fo[u].y, vz = sz + fo[u].z;
                    Ej = fmaxf(Ej, fmaxf(fabsf(vx), fmaxf(fabsf(vy), fabsf(vz))));
                }
                float* pa = reinterpret_cast<float*>(&S.sa[jj >> 1][e]) + (jj & 1);
                float* pz = reinterpret_cast<float*>(&S.sz[jj >> 1][e]) + (jj & 1);
                pa[0] = vx, pa[2] = vy, pz[0] = vz;
            }
            Ej = warp_fmax(Ej);
            PHASE(6);
            // coordinate errors: 2^-24 Ei (i side), 2^-23 (Ej + X) (cluster frame). The band
            // only widens with E, so thresholds computed for a running maximum of Ej stay
            // valid for later chunks: they are recomputed only when a chunk raises it.
            if (Ej > Ej_run) {
                Ej_run = fmaxf(Ej, Ej_run * 1.0625f);  // a little headroom: fewer recomputations
                const double ecoord = 5.9604644775390625e-08 * double(Ei) + 1.1920928955078125e-07 * (double(Ej_run) + double(Xo));
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const uint32_t k = lane + 32u * s;
                    float lo = -1.f, hi = -1.f;
                    if (ri[s] >= 0.0) {
                        const double rr2 = dmul(ri[s], ri[s]), g = guard_band(ri[s], rr2, ecoord);
                        lo = __double2float_rd(rr2 - g);
                        hi = __double2float_ru(rr2 + g);
                    }
                    S.ia[(k & 7) * 8 + (k >> 3)].w = lo, S.ihi[(k & 7) * 8 + (k >> 3)] = hi;
                }
                if (lane < nicl) S.pthr[lane] = __double2float_ru(pr2_me + guard_band(pr_me, pr2_me, ecoord));
                ecoord_cur = ecoord;
            }
            // symmetric: the pair radius is scale * max(h_i, h_j) = max(r_i, r_j) and the
            // prefilter radius scale * max(imaxh, jmaxh); lo/hi/thresholds are monotone in r,
            // so per-pair thresholds are the max of the per-particle ones
            float pthr_c = 0.f;
            if constexpr (SYM) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = uint32_t(u) * 4 + (lane >> 3), jj = lane & 7;
                    const uint32_t ce = __shfl_sync(0xffffffffu, cand, e);
                    const uint64_t j = uint64_t(ce) * cj + jj;
                    float lo = -1.f, hi = -1.f;
                    if (e < n && jj < cj && j < A.n) {
                        const double r = dmul(A.scale, A.h[j]), rr2 = dmul(r, r), g = guard_band(r, rr2, ecoord_cur);
                        lo = __double2float_rd(rr2 - g);
                        hi = __double2float_ru(rr2 + g);
                    }
                    if (e < n) {
                        reinterpret_cast<float*>(&S.sy.slo[jj >> 1][e])[jj & 1] = lo;
                        reinterpret_cast<float*>(&S.sy.shi[jj >> 1][e])[jj & 1] = hi;
                    }
                }
                if (valid) {
                    const double pr = dmul(A.scale, A.jgeo[cand].maxh), pr2 = dmul(pr, pr);
                    pthr_c = __double2float_ru(pr2 + guard_band(pr, pr2, ecoord_cur));
                }
            }
            if (lane < 32) S.cmask[lane] = 0;
            __syncwarp();
            // conservative fp32 prefilter, lane = candidate
            uint32_t pm = 0;
            if (valid) {
                float jlo[3] = {1e30f, 1e30f, 1e30f}, jhi[3] = {-1e30f, -1e30f, -1e30f};
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float4 a = S.sa[p][lane];
                    const auto z = S.sz[p][lane];
                    if (a.x != 1e30f) {
                        jlo[0] = fminf(jlo[0], a.x), jhi[0] = fmaxf(jhi[0], a.x);
                        jlo[1] = fminf(jlo[1], a.z), jhi[1] = fmaxf(jhi[1], a.z);
                        jlo[2] = fminf(jlo[2], z.x), jhi[2] = fmaxf(jhi[2], z.x);
                    }
                    if (a.y != 1e30f) {
                        jlo[0] = fminf(jlo[0], a.y), jhi[0] = fmaxf(jhi[0], a.y);
                        jlo[1] = fminf(jlo[1], a.w), jhi[1] = fmaxf(jhi[1], a.w);
                        jlo[2] = fminf(jlo[2], z.y), jhi[2] = fmaxf(jhi[2], z.y);
                    }
                }
                for (uint32_t b = 0; b < nicl; ++b) {
                    // half-list rule: the pair lives on the side whose i-cluster starts first (:133)
                    if (SYM && (icl_base + b) * 8 > uint64_t(cand) * cj) continue;
                    float s2 = 0.f;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const float g = fmaxf(fmaxf(S.iab[b][d], jlo[d]) - fminf(S.iab[b][3 + d], jhi[d]), 0.f);
                        s2 = fmaf(g, g, s2);
                    }
                    const float thr = SYM ? fmaxf(S.pthr[b], pthr_c) : S.pthr[b];
                    if (!(s2 > thr)) pm |= 1u << b;
                }
            }
            // items (b << 5 | c), candidate-major (one warp scan places each lane's set bits);
            // candidates overlapping the SC's own particles (i == j possible) last
            const bool self_me = valid && jl0 >= -7 && jl0 < kSC;
            const uint32_t npm = __popc(pm);
            const uint32_t c_ns = self_me ? 0u : npm, c_s = self_me ? npm : 0u;
            const uint32_t inc_ns = warp_incl_scan(c_ns), inc_s = warp_incl_scan(c_s);
            const uint32_t tot_ns = __shfl_sync(0xffffffffu, inc_ns, 31);
            const uint32_t nItems = tot_ns + __shfl_sync(0xffffffffu, inc_s, 31);
            {
                uint32_t at = self_me ? tot_ns + inc_s - c_s : inc_ns - c_ns;
                for (uint32_t m = pm; m; m &= m - 1) S.items[at++] = uint8_t(((__ffs(m) - 1) << 5) | lane);
            }
            __syncwarp();
            PHASE(7);
            // pair tests, one item per lane: hit iff some pair has d2 < lo (exact: d2 < r_i^2);
            // a row whose minimum lands in [lo, hi] is decided by the reference predicates
            for (uint32_t t0 = 0; t0 < nItems; t0 += 32) {
                const uint32_t t = t0 + lane;
                const bool iv = t < nItems;
                const uint32_t it8 = iv ? S.items[t] : 0u;
                const uint32_t c = it8 & 31u, b = it8 >> 5;
                const int j0 = __shfl_sync(0xffffffffu, jl0, c);
                const uint32_t cc = __shfl_sync(0xffffffffu, cand, c);
                const bool self = iv && j0 >= -7 && j0 < kSC;
                ulonglong2 Ja[4];
                ulonglong2 Jz[4];  // {z pair, -} (16-byte staging rows measured faster than 8-byte ones)
                float2 Jlo[4], Jhi[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    Ja[p] = reinterpret_cast<const ulonglong2&>(S.sa[p][c]);
                    Jz[p].x = reinterpret_cast<const f2&>(S.sz[p][c]);
                    if constexpr (SYM) Jlo[p] = S.sy.slo[p][c], Jhi[p] = S.sy.shi[p][c];
                }
                bool hit = false;
                uint32_t band_rows = 0;
                auto rows = [&](auto SELF) {
                    constexpr bool kSelf = decltype(SELF)::value;
#pragma unroll 1
                    for (int ii = 0; ii < 8 && iv && !hit; ++ii) {
                        const float4 I = S.ia[ii * 8 + b];
                        const f2 xi2 = f2p(I.x, I.x), yi2 = f2p(I.y, I.y), zi2 = f2p(I.z, I.z);
                        const int iself = kSelf && self ? int(b * 8 + ii) - j0 : -1;
                        float mn = 3.0e38f, mh = 3.0e38f;
                        const float hii = S.ihi[ii * 8 + b];
#pragma unroll
                        for (int p = 0; p < 4; ++p) {
                            float d2a, d2b;
                            const f2 dx = f2sub(xi2, Ja[p].x), dy = f2sub(yi2, Ja[p].y), dz = f2sub(zi2, Jz[p].x);
                            f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                            if (kSelf) {
                                if (iself == 2 * p) d2a = 3.0e38f;
                                if (iself == 2 * p + 1) d2b = 3.0e38f;
                            }
                            if (SYM) {  // margins to the per-pair thresholds max(lo_i, lo_j), max(hi_i, hi_j)
                                mn = fminf(mn, fminf(d2a - fmaxf(I.w, Jlo[p].x), d2b - fmaxf(I.w, Jlo[p].y)));
                                mh = fminf(mh, fminf(d2a - fmaxf(hii, Jhi[p].x), d2b - fmaxf(hii, Jhi[p].y)));
                            } else {
                                mn = fminf(mn, fminf(d2a, d2b));
                            }
                        }
                        if (SYM) {
                            if (mn < 0.f) hit = true;
                            else if (mh <= 0.f) band_rows |= 1u << ii;
                        } else {
                            if (mn < I.w) hit = true;
                            else if (mn <= hii) band_rows |= 1u << ii;
                        }
                    }
                };
                if (__any_sync(0xffffffffu, self)) rows(BoolC<true>());
                else rows(BoolC<false>());
                if (SFCNL_UNLIKELY(iv && !hit && band_rows)) hit = band_item<SYM>(A, p0, icl_base, b, cc, band_rows);
                if (iv && hit) atomicOr(&S.cmask[c], 1u << b);
            }
            __syncwarp();
            PHASE(8);
            mask = valid ? S.cmask[lane] : 0u;
        }
        // ordered compaction of the chunk's entries with mask != 0
        const bool keep = valid && mask != 0;
        const unsigned kb = __ballot_sync(0xffffffffu, keep);
        if (nE + __popc(kb) > Sm::kE) return false;
        if (keep) {
            const uint32_t at = nE + __popc(kb & lanemask_lt());
            S.eidx[at] = A.lc2g ? A.lc2g[cand] : cand, S.emsk[at] = uint8_t(mask);
        }
        nE += __popc(kb);
        __syncwarp();  // staging consumed
    }
    __syncwarp();

    PHASE(3);
    // ---- 5b. serialization (neighbor_build.cpp:164-182): masks, then the index list
    uint8_t* ebuf = S.u.ebuf;
    const uint32_t mbytes = nE;  // one mask byte per entry (ci == 8)
    if (mbytes + 4 > Sm::kB) return false;
    for (uint32_t k = lane; k < nE; k += 32) ebuf[k] = S.emsk[k];
    uint32_t pos = mbytes;
    if (!A.compress) {
        if (mbytes + 4 * nE > Sm::kB) return false;
        for (uint32_t k = lane; k < nE; k += 32) {
            const uint32_t v = S.eidx[k];
#pragma unroll
            for (int b = 0; b < 4; ++b) ebuf[mbytes + 4 * k + b] = uint8_t(v >> (8 * b));
        }
        __syncwarp();  // the byte stores are read back as words by the copy-out below
        pos = mbytes + 4 * nE;
    } else {
        // nibble codec (nibble_codec.cpp:56-134): blocks of w differences
        const uint32_t w = uint32_t(A.w);
        for (uint32_t bb = 0; bb < nE; bb += w) {
            const uint32_t len = min(w, nE - bb);
            uint64_t dv[2];
            uint32_t nd[2], isset[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const uint32_t k = lane + 32u * s;
                dv[s] = 1, nd[s] = 0, isset[s] = 0;
                if (k < len && (s == 0 || w == 64)) {
                    const uint64_t cur = S.eidx[bb + k];
                    dv[s] = (bb + k == 0) ? cur + 1 : cur - uint64_t(S.eidx[bb + k - 1]);
                    isset[s] = dv[s] != 1;
                    nd[s] = (dv[s] > 9) ? uint32_t(nibble_count(dv[s])) : 0u;
                }
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, isset[0]);
            const unsigned m1 = __ballot_sync(0xffffffffu, isset[1]);
            const uint32_t ninfo = __popc(m0) + __popc(m1);
            const uint32_t inc0 = warp_incl_scan(nd[0]);
            const uint32_t tot0 = __shfl_sync(0xffffffffu, inc0, 31);
            const uint32_t inc1 = warp_incl_scan(nd[1]);
            const uint32_t nib = ninfo + tot0 + __shfl_sync(0xffffffffu, inc1, 31);
            const uint32_t bsize = w / 8 + (nib + 1) / 2;
            if (pos + bsize > Sm::kB) return false;
            const unsigned long long bm = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
            if (lane < w / 8) ebuf[pos + lane] = uint8_t(bm >> (8 * lane));
            for (uint32_t q = lane; q < (nib + 1) / 2; q += 32) ebuf[pos + w / 8 + q] = 0;
            __syncwarp();
            const uint32_t nbase = (pos + w / 8) * 2;  // nibble index of the block's first nibble
            unsigned int* words = reinterpret_cast<unsigned int*>(ebuf);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                if (!isset[s]) continue;
                const uint32_t info_at = s == 0 ? __popc(m0 & lanemask_lt()) : __popc(m0) + __popc(m1 & lanemask_lt());
                const uint64_t v = dv[s];
                const uint32_t infov = v <= 9 ? uint32_t(v + 6) : nd[s] - 1;
                uint32_t t = nbase + info_at;
                atomicOr(&words[t >> 3], infov << (4 * (t & 7)));
                if (nd[s]) {
                    uint32_t dstart = ninfo + (s == 0 ? inc0 - nd[0] : tot0 + inc1 - nd[1]);
                    for (int p = int(nd[s]) - 1; p >= 0; --p, ++dstart) {
                        t = nbase + dstart;
                        atomicOr(&words[t >> 3], uint32_t((v >> (4 * p)) & 15u) << (4 * (t & 7)));
                    }
                }
            }
            __syncwarp();
            pos += bsize;
        }
    }
    const uint32_t size = pos;

    PHASE(4);
    // ---- publish: bump-allocate the scratch and copy
    unsigned long long off = 0;
    if (lane == 0) {
        const unsigned long long need = (size + 15ull) & ~15ull;
        off = atomicAdd(&A.ctl[0], need);
        if (off + need > A.scratch_cap) {
            A.ctl[2] = 1;
            off = ~0ull;
        }
        A.counts[sc] = nE;
        A.sizes[sc] = size;
        A.soff[sc] = off;
    }
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off != ~0ull) {
        const unsigned int* src = reinterpret_cast<const unsigned int*>(ebuf);
        unsigned int* dst = reinterpret_cast<unsigned int*>(A.scratch + off);
        for (uint32_t q = lane; q < (size + 3) / 4; q += 32) dst[q] = src[q];
    }
    __syncwarp();
    PHASE(5);
    return true;
}

// list == nullptr: SCs [sc_begin, sc_end) (main tier); else the `count` SCs of list
// (overflow re-run). SCs beyond this tier's capacity go to overflow_out / ctl[ctl_slot].
template <class Sm, int MINB>
__global__ void __launch_bounds__(kBwWarps * 32, MINB) k_build_warp(const __grid_constant__ BuildArgs A, uint64_t sc_begin,
                                                                     uint64_t sc_end, unsigned long long* __restrict__ work,
                                                                     const uint32_t* __restrict__ list,
                                                                     uint32_t* __restrict__ overflow_out, int ctl_slot) {
    extern __shared__ __align__(16) unsigned char dsm[];
    Sm& S = reinterpret_cast<Sm*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (sc_begin + t >= sc_end) break;
        const uint64_t sc = list ? uint64_t(list[t]) : sc_begin + t;
        if (!build_sc_warp(A, S, sc)) {
            if (lane == 0) {
                const unsigned long long slot = atomicAdd(&A.ctl[ctl_slot], 1ull);
                overflow_out[slot] = uint32_t(sc);
                A.counts[sc] = 0, A.sizes[sc] = 0, A.soff[sc] = 0;
            }
        }
        __syncwarp();
    }
}

// Halo marking for a domain decomposition: the candidate j-clusters of
// the range's SCs, i.e. the clusters of every leaf the build's traversal accepts, are
// flagged. Warp per SC (same BFS as the build); SCs whose frontier overflows are
// listed for the global-memory fallback (k_halo_global).
__global__ void __launch_bounds__(256) k_halo_warp(const __grid_constant__ BuildArgs A, uint64_t sc_begin, uint64_t sc_end,
                                                   uint8_t* __restrict__ jflags, unsigned long long* __restrict__ work) {
    __shared__ uint32_t fr[8][2 * kBwF];
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        const uint64_t sc = sc_begin + __shfl_sync(0xffffffffu, t, 0);
        if (sc >= sc_end) break;
        const uint64_t icl_base = sc * A.icl_per_sc;
        const uint32_t nicl = uint32_t(tmin<uint64_t>(icl_base + A.icl_per_sc, A.num_icl) - icl_base);
        Geo scg;
        double r2;
        sc_box(A, icl_base, nicl, scg, r2);
        uint32_t* fa;
        const uint32_t nA = warp_bfs(A, scg, r2, fr[w], fr[w] + kBwF, &fa);
        if (nA == ~0u) {
            if (lane == 0) {
                const unsigned long long slot = atomicAdd(&A.ctl[1], 1ull);
                A.overflow_list[slot] = uint32_t(sc);
                if (A.leaf_count) A.leaf_count[sc - A.leaf_sc0] = ~0u;
            }
            __syncwarp();
            continue;
        }
        for (uint32_t k = lane; k < nA; k += 32) {
            const Node nd = A.nodes[fa[k] & ~kTag];
            if (jflags)
                for (uint32_t j = nd.pbegin / A.cj; j <= (nd.pend - 1) / A.cj; ++j) jflags[j] = 1;
            if (A.leaf_cache && nA <= kLeafCacheCap) A.leaf_cache[(sc - A.leaf_sc0) * kLeafCacheCap + k] = fa[k];
        }
        if (A.leaf_count && lane == 0) A.leaf_count[sc - A.leaf_sc0] = nA <= kLeafCacheCap ? nA : ~0u;
        __syncwarp();
    }
}
