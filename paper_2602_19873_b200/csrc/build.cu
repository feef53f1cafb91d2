// (2)(3)(4) Neighbor-list build: per-super-cluster traversal, interaction masks
// and nibble-codec encode, then a size scan and a compaction into the final blob.
//
// Replaces build_neighbor_store (neighbor_build.cpp:74-184) including
// collect_candidates (:43-65), the mask loop (:128-161) and the serial
// serialization + codec::encode (:164-182, nibble_codec.cpp:117-134).
//
// One CTA (128 threads) per super-cluster (SC, 64 particles):
//  * traversal: level-synchronous BFS over the octree with an ORDERED frontier in
//    shared memory (stable block-scan compaction keeps key order; accepted leaves
//    ride along tagged). A node is accepted iff non-empty and
//    aabb_dist_sq(sc_aabb, node_aabb) <= r^2 (bit-exact fp64, common.cuh). Because
//    node boxes nest and aabb_dist_sq is monotone under containment, BFS accepts
//    exactly the leaves the reference's DFS accepts, in the same key order.
//  * candidates: union of the accepted leaves' j-cluster ranges, deduplicated
//    against the previous leaf exactly like `out.back() != j` (:57-58).
//  * masks: one thread per candidate j-cluster runs the reference loop for its 8
//    i-clusters: half-list rule (symmetric), AABB prefilter, exact pair test with
//    early exit -- all predicates in round-to-nearest fp64.
//  * encode: entries with mask != 0 are compacted in order; masks are written
//    little-endian, the index list is delta/nibble encoded one 32/64-wide block at
//    a time by warp 0 (ballot for the block mask, warp scans for nibble offsets,
//    smem atomicOr to pack nibbles low-first).
//  * the SC's bytes go to a bump-allocated scratch area; a u32->u64 scan of the
//    per-SC sizes gives NeighborStore::offsets and a warp-per-SC copy builds the blob.
// SCs whose frontier/candidates/bytes exceed the shared-memory capacities are
// re-run by the same code with global-memory workspaces (fallback launch).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "ctx.hpp"
#include "scan.hpp"

namespace sfcnl_cu {
namespace {

constexpr int kBuildThreads = 128;
constexpr uint32_t kTag = 0x80000000u;
constexpr uint32_t kFCap = 1024, kCCap = 1024, kECap = 8192;

struct BuildArgs {
    uint64_t n;
    Box box;
    double scale;
    uint32_t ci, cj, icl_per_sc, mask_bytes;
    int w, compress, symmetric;
    uint64_t num_icl;
    const double* x;
    const double* y;
    const double* z;
    const double* h;
    const Node* nodes;
    const Geo* ngeo;
    const float4* ngeo32;      // node boxes rounded to fp32 {lo, -}, {hi, -} (gather traversal pre-test), or null
    float trav_m;              // max |coordinate| of a (shifted) box bound, for the pre-test's error bound
    const Geo* igeo;
    const Geo* jgeo;
    uint32_t* counts;
    uint32_t* sizes;
    uint64_t* soff;
    uint8_t* scratch;
    unsigned long long* ctl;  // [0] scratch top, [1] overflow count, [2] scratch overflow flag, [3] max h bits, [4] medium-tier overflow count
    uint64_t scratch_cap;
    uint32_t* overflow_list;
    const float4* frame;       // cluster-frame staging copy (frame.cu)
    const unsigned* frame_x;   // its max |offset| per axis (float bits)
    unsigned long long* prof;  // phase clocks (SFCNL_PHASE_PROF builds)
    uint32_t* leaf_cache;      // accepted leaves per SC of [sc_lo, ...) (halo_mark -> range build), or null
    uint32_t* leaf_count;      // their number per SC (~0u: not cached)
    uint64_t leaf_sc0;         // first SC of the cache
    const uint32_t* lc2g;      // domain decomposition (dd.cu): local cluster -> global id of the encoded list, or null
    DevError* err;
};

struct Workspace {
    uint32_t* fa;
    uint32_t* fb;
    uint32_t* cand;
    unsigned long long* cmask;
    uint8_t* ebuf;
    uint32_t fcap, ccap, ecap;
    bool fast;  // shared-memory workspace: the fast mask path may run
};

__device__ __forceinline__ int nibble_count(uint64_t v) { return (64 - __clzll(v) + 3) / 4; }

typedef unsigned long long f2;  // packed fp32 pair for FADD2/FFMA2/FMUL2
__device__ __forceinline__ f2 f2p(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2u(f2 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2 f2sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2fma(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Rounding-error guard on a squared distance computed in fp32 from coordinates
// relative to a common origin (each coordinate within 2^-24 * E of its fp64 value):
// |d2_f32 - d2| <= 3*2^-24*r2 + 3.5*r*ex + 3*ex^2 near d2 ~ r2, ex = 2^-23*E + 2^-24*r.
__device__ __forceinline__ double d2_guard(double r, double r2, float E) {
    const double ex = 1.1920928955078125e-07 * double(E) + 5.9604644775390625e-08 * r;
    return 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
}

// Exact pair test of one (i, j) in reference arithmetic (neighbor_build.cpp:140-155).
__device__ __noinline__ bool exact_hit(const BuildArgs& A, double xi, double yi, double zi, double hi,
                                       uint64_t j) {
    const double rr = dmul(A.scale, A.symmetric ? smax(hi, A.h[j]) : hi);
    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, nullptr, nullptr, nullptr);
    return d2 <= dmul(rr, rr);
}

#include "build_fast.cuh"
#include "build_warp.cuh"
#include "build_p1.cuh"

// Ordered-frontier BFS over the octree for one SC (collect_candidates,
// neighbor_build.cpp:43-65). Leaves the accepted leaves (tagged, key order) in
// *front and returns their number, or ~0u when the frontier exceeds W.fcap.
__device__ __forceinline__ uint32_t sc_traverse(const BuildArgs& A, const Workspace& W, const Geo& scg,
                                                double r2, uint32_t* scratch, int* s_flag, uint32_t** front) {
    const unsigned tid = threadIdx.x;
    uint32_t* fa = W.fa;
    uint32_t* fb = W.fb;
    if (tid == 0) fa[0] = 0;
    uint32_t nA = 1;
    for (;;) {
        uint32_t nB = 0;
        if (tid == 0) *s_flag = 0;
        __syncthreads();
        for (uint32_t base = 0; base < nA; base += blockDim.x) {
            const uint32_t k = base + tid;
            uint32_t emit = 0, e = 0;
            int32_t fc = -1;
            if (k < nA) {
                e = fa[k];
                if (e & kTag) {
                    emit = 1;
                } else {
                    const Node nd = A.nodes[e];
                    if (nd.pend > nd.pbegin) {
                        const Geo ng = A.ngeo[e];
                        double rr2 = r2;
                        if (A.symmetric) {
                            const double rr = dmul(A.scale, smax(scg.maxh, ng.maxh));
                            rr2 = dmul(rr, rr);
                        }
                        if (!(aabb_dist_sq(scg, ng, A.box) > rr2)) {
                            fc = nd.first_child;
                            emit = fc < 0 ? 1 : 8;
                        }
                    }
                }
            }
            uint32_t tot;
            const uint32_t ex = block_excl_scan(emit, scratch, &tot);
            if (nB + tot > W.fcap) {
                __syncthreads();
                return ~0u;
            }
            if (emit == 1) fb[nB + ex] = (e & kTag) ? e : (e | kTag);
            if (emit == 8) {
                for (int c = 0; c < 8; ++c) fb[nB + ex + c] = uint32_t(fc + c);
                *s_flag = 1;
            }
            nB += tot;
        }
        __syncthreads();
        uint32_t* t = fa;
        fa = fb, fb = t;
        nA = nB;
        if (!*s_flag) break;
        __syncthreads();
    }
    *front = fa;
    return nA;
}

// SC geometry = union of its i-clusters (neighbor_build.cpp:113-118); thread 0.
__device__ __forceinline__ void sc_geometry(const BuildArgs& A, const Geo* s_igeo, uint32_t nicl, Geo* s_sc,
                                            double* s_r2) {
    Geo g;
    geo_init(g);
    for (uint32_t b = 0; b < nicl; ++b) {
        geo_extend(g, s_igeo[b]);
        g.maxh = smax(g.maxh, s_igeo[b].maxh);
    }
    *s_sc = g;
    const double r = dmul(A.scale, g.maxh);
    *s_r2 = dmul(r, r);
}

// Returns false on capacity overflow (caller re-runs the SC in global-memory mode).
__device__ bool build_sc(const BuildArgs& A, const Workspace& W, uint64_t sc) {
    __shared__ Geo s_igeo[64];
    __shared__ double s_x[64], s_y[64], s_z[64], s_h[64];
    __shared__ Geo s_sc;
    __shared__ double s_r2;
    __shared__ uint32_t scratch[33];
    __shared__ int s_flag;
    __shared__ uint32_t s_n[2];
    const unsigned tid = threadIdx.x;
    const uint64_t n = A.n;
    const uint64_t icl_base = sc * A.icl_per_sc;
    const uint64_t icl_end = tmin<uint64_t>(icl_base + A.icl_per_sc, A.num_icl);
    const uint32_t nicl = uint32_t(icl_end - icl_base);
    const uint64_t p0 = sc * kSC;
    const uint32_t np = uint32_t(tmin<uint64_t>(p0 + kSC, n) - p0);
    for (uint32_t b = tid; b < nicl; b += blockDim.x) s_igeo[b] = A.igeo[icl_base + b];
    for (uint32_t k = tid; k < np; k += blockDim.x) {
        s_x[k] = A.x[p0 + k], s_y[k] = A.y[p0 + k], s_z[k] = A.z[p0 + k], s_h[k] = A.h[p0 + k];
    }
    __syncthreads();
    if (tid == 0) sc_geometry(A, s_igeo, nicl, &s_sc, &s_r2);
    __syncthreads();
    const Geo scg = s_sc;
    const double r2 = s_r2;

    // ---- traversal (collect_candidates, neighbor_build.cpp:43-65)
    uint32_t* fa;
    const uint32_t nA = sc_traverse(A, W, scg, r2, scratch, &s_flag, &fa);
    if (nA == ~0u) return false;

    // ---- candidate j-clusters (union of accepted leaf ranges, in order)
    uint32_t nC = 0;
    for (uint32_t base = 0; base < nA; base += blockDim.x) {
        const uint32_t k = base + tid;
        uint32_t cnt = 0, start = 0;
        if (k < nA) {
            const Node nd = A.nodes[fa[k] & ~kTag];
            const uint32_t f = nd.pbegin / A.cj, l = (nd.pend - 1) / A.cj;
            start = f;
            if (k > 0) {
                const Node pv = A.nodes[fa[k - 1] & ~kTag];
                if ((pv.pend - 1) / A.cj == f) start = f + 1;
            }
            cnt = l + 1 - start;
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan(cnt, scratch, &tot);
        if (nC + tot > W.ccap) {
            __syncthreads();
            return false;
        }
        for (uint32_t j = 0; j < cnt; ++j) W.cand[nC + ex + j] = start + j;
        nC += tot;
    }
    __syncthreads();

    // ---- interaction masks (neighbor_build.cpp:128-161)
    const bool fast = W.fast && A.ci == 8 && (A.cj == 8 || A.cj == 4) && !A.symmetric &&
                      fast_masks(A, W, nC, nicl, p0, np, s_x, s_y, s_z, s_h, s_igeo);
    for (uint32_t c = tid; c < nC && !fast; c += blockDim.x) {
        const uint32_t jcl = W.cand[c];
        const Geo jg = A.jgeo[jcl];
        const uint64_t jb = uint64_t(jcl) * A.cj, je = tmin<uint64_t>(jb + A.cj, n);
        unsigned long long mask = 0;
        for (uint32_t b = 0; b < nicl; ++b) {
            const uint64_t gi = icl_base + b;
            if (A.symmetric && gi * A.ci > jb) continue;
            const double pre_r =
                dmul(A.scale, A.symmetric ? smax(s_igeo[b].maxh, jg.maxh) : s_igeo[b].maxh);
            if (aabb_dist_sq(s_igeo[b], jg, A.box) > dmul(pre_r, pre_r)) continue;
            const uint64_t ib = gi * A.ci, ie = tmin<uint64_t>(ib + A.ci, n);
            bool hit = false;
            for (uint64_t i = ib; i < ie && !hit; ++i) {
                const uint32_t li = uint32_t(i - p0);
                const double xi = s_x[li], yi = s_y[li], zi = s_z[li], hi = s_h[li];
                for (uint64_t j = jb; j < je; ++j) {
                    if (i == j) continue;
                    const double hj = A.symmetric ? __ldg(A.h + j) : 0.0;
                    const double rr = dmul(A.scale, A.symmetric ? smax(hi, hj) : hi);
                    const double d2 = pair_d2_exact(xi, yi, zi, __ldg(A.x + j), __ldg(A.y + j),
                                                    __ldg(A.z + j), A.box, nullptr, nullptr, nullptr);
                    if (d2 <= dmul(rr, rr)) {
                        hit = true;
                        break;
                    }
                }
            }
            if (hit) mask |= 1ull << b;
        }
        W.cmask[c] = mask;
    }
    __syncthreads();

    // ---- ordered compaction of entries with mask != 0
    uint32_t nE = 0;
    for (uint32_t base = 0; base < nC; base += blockDim.x) {
        const uint32_t k = base + tid;
        const bool keep = k < nC && W.cmask[k] != 0;
        const uint32_t jc = keep ? W.cand[k] : 0;
        const unsigned long long mk = keep ? W.cmask[k] : 0;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(keep ? 1u : 0u, scratch, &tot);
        if (keep) W.cand[nE + ex] = A.lc2g ? A.lc2g[jc] : jc, W.cmask[nE + ex] = mk;
        nE += tot;
        __syncthreads();
    }

    // ---- serialization (neighbor_build.cpp:164-182)
    const uint32_t mbytes = nE * A.mask_bytes;
    if (mbytes + 4 > W.ecap) {
        __syncthreads();
        return false;
    }
    for (uint32_t k = tid; k < nE; k += blockDim.x)
        for (uint32_t b = 0; b < A.mask_bytes; ++b) W.ebuf[k * A.mask_bytes + b] = uint8_t(W.cmask[k] >> (8 * b));
    uint32_t size = mbytes;
    if (!A.compress) {
        size = mbytes + 4 * nE;
        if (size > W.ecap) {
            __syncthreads();
            return false;
        }
        for (uint32_t k = tid; k < nE; k += blockDim.x)
            for (int b = 0; b < 4; ++b) W.ebuf[mbytes + 4 * k + b] = uint8_t(W.cand[k] >> (8 * b));
    } else if (tid < 32) {
        // nibble codec (nibble_codec.cpp:56-134): blocks of w differences
        const unsigned lane = tid;
        const uint32_t w = uint32_t(A.w);
        uint32_t pos = mbytes;
        bool over = false;
        for (uint32_t bb = 0; bb < nE && !over; bb += w) {
            const uint32_t len = min(w, nE - bb);
            uint64_t dv[2];
            uint32_t nd[2], isset[2];
            uint32_t data_total = 0;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const uint32_t k = lane + 32u * s;
                dv[s] = 1, nd[s] = 0, isset[s] = 0;
                if (k < len && (s == 0 || w == 64)) {
                    const uint64_t cur = W.cand[bb + k];
                    dv[s] = (bb + k == 0) ? cur + 1 : cur - uint64_t(W.cand[bb + k - 1]);
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
            data_total = tot0 + __shfl_sync(0xffffffffu, inc1, 31);
            const uint32_t nib = ninfo + data_total;
            const uint32_t bsize = w / 8 + (nib + 1) / 2;
            if (pos + bsize > W.ecap) {
                over = true;
                break;
            }
            // block mask bytes, then zero the nibble bytes of this block
            const unsigned long long bm = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
            if (lane < w / 8) W.ebuf[pos + lane] = uint8_t(bm >> (8 * lane));
            for (uint32_t q = lane; q < (nib + 1) / 2; q += 32) W.ebuf[pos + w / 8 + q] = 0;
            __syncwarp();
            const uint32_t nbase = (pos + w / 8) * 2;  // nibble index of the block's first nibble
            unsigned int* words = reinterpret_cast<unsigned int*>(W.ebuf);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                if (!isset[s]) continue;
                const uint32_t k = lane + 32u * s;
                const uint32_t info_at =
                    s == 0 ? __popc(m0 & ((1u << lane) - 1u)) : __popc(m0) + __popc(m1 & ((1u << lane) - 1u));
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
                (void)k;
            }
            __syncwarp();
            pos += bsize;
        }
        if (lane == 0) {
            s_n[0] = pos;
            s_n[1] = over ? 1u : 0u;
        }
    }
    __syncthreads();
    if (A.compress) {
        if (s_n[1]) {
            __syncthreads();
            return false;
        }
        size = s_n[0];
    }

    // ---- publish: bump-allocate scratch and copy
    __shared__ unsigned long long s_off;
    if (tid == 0) {
        const unsigned long long need = (size + 15ull) & ~15ull;
        const unsigned long long off = atomicAdd(&A.ctl[0], need);
        if (off + need > A.scratch_cap) {
            A.ctl[2] = 1;
            s_off = ~0ull;
        } else {
            s_off = off;
        }
        A.counts[sc] = nE;
        A.sizes[sc] = size;
        A.soff[sc] = s_off;
    }
    __syncthreads();
    if (s_off != ~0ull) {
        const uint32_t words = (size + 3) / 4;
        const unsigned int* src = reinterpret_cast<const unsigned int*>(W.ebuf);
        unsigned int* dst = reinterpret_cast<unsigned int*>(A.scratch + s_off);
        for (uint32_t q = tid; q < words; q += blockDim.x) dst[q] = src[q];
    }
    __syncthreads();
    return true;
}

__global__ void __launch_bounds__(kBuildThreads, 5) k_build_smem(const __grid_constant__ BuildArgs A, uint64_t sc_begin, uint64_t sc_end) {
    // region0 is used in turn by the traversal frontier (fa|fb) and the encoder's bytes.
    static_assert(kECap <= 2 * kFCap * 4, "region0 size");
    __shared__ __align__(16) uint32_t region0[2 * kFCap];
    __shared__ uint32_t cand[kCCap];
    __shared__ unsigned long long cmask[kCCap];
    const Workspace W{region0, region0 + kFCap, cand, cmask, reinterpret_cast<uint8_t*>(region0),
                      kFCap, kCCap, kECap, true};
    for (uint64_t sc = sc_begin + blockIdx.x; sc < sc_end; sc += gridDim.x) {
        if (!build_sc(A, W, sc)) {
            if (threadIdx.x == 0) {
                const unsigned long long slot = atomicAdd(&A.ctl[1], 1ull);
                A.overflow_list[slot] = uint32_t(sc);
                A.counts[sc] = 0, A.sizes[sc] = 0, A.soff[sc] = 0;
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kBuildThreads) k_build_global(const __grid_constant__ BuildArgs A, const uint32_t* list,
                                                                 uint64_t count, uint8_t* ws,
                                                                 uint64_t ws_stride, uint32_t fcap,
                                                                 uint32_t ccap, uint32_t ecap) {
    uint8_t* base = ws + blockIdx.x * ws_stride;
    Workspace W;
    W.fa = reinterpret_cast<uint32_t*>(base);
    W.fb = W.fa + fcap;
    W.cand = W.fb + fcap;
    W.cmask = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(W.cand + ccap) + 15) & ~uintptr_t(15));
    W.ebuf = reinterpret_cast<uint8_t*>(W.cmask + ccap);
    W.fcap = fcap, W.ccap = ccap, W.ecap = ecap;
    W.fast = true;  // global-memory workspaces; the fp32 guard-band masks still apply
    for (uint64_t t = blockIdx.x; t < count; t += gridDim.x) {
        const uint64_t sc = list[t];
        if (!build_sc(A, W, sc)) {
            if (threadIdx.x == 0) raise_error(A.err, sc, SFCNL_BUILD_ERROR, 3, 0);
            __syncthreads();
        }
    }
}

// ---- halo marking (domain decomposition) -------------------------
// The particles a rank's build and pass read outside its own range are exactly the
// candidate j-clusters of its SCs (accepted leaves' cluster ranges). One CTA per SC
// runs the build's traversal and flags those clusters.
__device__ bool halo_sc(const BuildArgs& A, const Workspace& W, uint64_t sc, uint8_t* jflags) {
    __shared__ Geo s_igeo[64];
    __shared__ Geo s_sc;
    __shared__ double s_r2;
    __shared__ uint32_t scratch[33];
    __shared__ int s_flag;
    const unsigned tid = threadIdx.x;
    const uint64_t icl_base = sc * A.icl_per_sc;
    const uint64_t icl_end = tmin<uint64_t>(icl_base + A.icl_per_sc, A.num_icl);
    const uint32_t nicl = uint32_t(icl_end - icl_base);
    for (uint32_t b = tid; b < nicl; b += blockDim.x) s_igeo[b] = A.igeo[icl_base + b];
    __syncthreads();
    if (tid == 0) sc_geometry(A, s_igeo, nicl, &s_sc, &s_r2);
    __syncthreads();
    uint32_t* fa;
    const uint32_t nA = sc_traverse(A, W, s_sc, s_r2, scratch, &s_flag, &fa);
    if (nA == ~0u) return false;
    for (uint32_t k = tid; k < nA; k += blockDim.x) {
        const Node nd = A.nodes[fa[k] & ~kTag];
        for (uint32_t j = nd.pbegin / A.cj; j <= (nd.pend - 1) / A.cj; ++j) jflags[j] = 1;
    }
    __syncthreads();
    return true;
}

__global__ void __launch_bounds__(kBuildThreads) k_halo_global(const __grid_constant__ BuildArgs A, const uint32_t* list, uint64_t count,
                                                               uint32_t* ws, uint32_t fcap, uint8_t* jflags) {
    uint32_t* base = ws + uint64_t(blockIdx.x) * 2 * fcap;
    const Workspace W{base, base + fcap, nullptr, nullptr, nullptr, fcap, 0, 0, false};
    for (uint64_t t = blockIdx.x; t < count; t += gridDim.x) halo_sc(A, W, list[t], jflags);
}

__global__ void k_compact(uint64_t num_sc, const uint32_t* __restrict__ sizes,
                          const uint64_t* __restrict__ soff, const uint64_t* __restrict__ offsets,
                          const uint8_t* __restrict__ scratch, uint8_t* __restrict__ blob) {
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    if (warp >= num_sc) return;
    const uint32_t sz = sizes[warp];
    const uint8_t* src = scratch + soff[warp];
    uint8_t* dst = blob + offsets[warp];
    for (uint32_t k = lane_id(); k < sz; k += 32) dst[k] = src[k];
}

// validate (core.hpp:201-216) + max h for the periodic precondition.
__global__ void k_validate(uint64_t n, const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, const double* __restrict__ h, Box box,
                           unsigned long long* maxh_bits, DevError* err) {
    unsigned long long local = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double hv = h[i];
        const double p[3] = {x[i], y[i], z[i]};
        if (!(hv > 0)) {
            raise_error(err, i, SFCNL_INPUT_ERROR, 1, 0);
            continue;
        }
        for (int d = 0; d < 3; ++d) {
            if (!isfinite(p[d])) {
                raise_error(err, i, SFCNL_INPUT_ERROR, 2, 0);
                break;
            }
            if (p[d] < box.lo[d] || p[d] > box.hi[d]) {
                raise_error(err, i, SFCNL_INPUT_ERROR, 3, 0);
                break;
            }
        }
        local = max(local, (unsigned long long)__double_as_longlong(hv));  // h > 0: order-preserving
    }
    for (int o = 16; o > 0; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
    if (lane_id() == 0 && local) atomicMax(maxh_bits, local);
}

#ifndef SFCNL_TRAV_CTAS
#define SFCNL_TRAV_CTAS 6
#endif
constexpr int kTravCtas = SFCNL_TRAV_CTAS;  // CTAs (8 warps) per SM of the traversal kernel

// Node boxes rounded to nearest fp32 for the traversal's pre-test (build_warp.cuh).
__global__ void k_node_box32(uint64_t m, const Geo* __restrict__ g, float4* __restrict__ out) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < m; k += uint64_t(gridDim.x) * blockDim.x) {
        const Geo v = g[k];
        out[2 * k] = make_float4(float(v.lo[0]), float(v.lo[1]), float(v.lo[2]), 0.f);
        out[2 * k + 1] = make_float4(float(v.hi[0]), float(v.hi[1]), float(v.hi[2]), 0.f);
    }
}

// fp32 node boxes for the gather traversal (null for symmetric stores or when disabled)
int node_boxes32(sfcnl_cu_ctx* c, BuildArgs& A, bool gather) {
    A.ngeo32 = nullptr;
    A.trav_m = 0.f;
    if (!gather || getenv("SFCNL_TRAV_FP64") || c->num_nodes == 0) return 0;
    SFCNL_CUDA_TRY(c->node_geo32.reserve(c->num_nodes * 2 * sizeof(float4)));
    launch(c, k_node_box32, dim3(unsigned(std::min<uint64_t>((c->num_nodes + 255) / 256, uint64_t(c->num_sms) * 8))),
           dim3(256), 0, uint64_t(c->num_nodes), (const Geo*)A.ngeo, c->node_geo32.as<float4>());
    A.ngeo32 = c->node_geo32.as<const float4>();
    double m = 0.0;
    for (int d = 0; d < 3; ++d)
        m = std::max(m, std::max(std::fabs(A.box.lo[d]), std::fabs(A.box.hi[d])) + (A.box.per[d] ? A.box.len[d] : 0.0));
    A.trav_m = float(m * 1.0001);
    return 0;
}

// Main warp-build tier over [sc0, sc1), then the medium tier over its overflow list;
// SCs beyond both are returned in (*ovf_list, *ovf_count) for k_build_global.
template <class Sm, class SmM>
int launch_build_warp(sfcnl_cu_ctx* c, const BuildArgs& A, uint64_t sc0, uint64_t sc1, uint64_t num_sc,
                      unsigned long long* ctl, const uint32_t** ovf_list, unsigned long long* ovf_count) {
    constexpr int kMinMain = sizeof(Sm) * kBwWarps * 6 + 6 * 1024 <= 228 * 1024 ? 6 : (sizeof(Sm) * kBwWarps * 5 <= 227 * 1024 ? 5 : 4);
    const size_t smem = size_t(kBwWarps) * sizeof(Sm);
    cudaFuncSetAttribute(k_build_warp<Sm, kMinMain>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
    const unsigned grid = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>((num_sc + kBwWarps - 1) / kBwWarps, uint64_t(c->num_sms) * kMinMain)));
    launch(c, k_build_warp<Sm, kMinMain>, dim3(grid), dim3(kBwWarps * 32), smem, A, sc0, sc1,
           c->work_ctr.as<unsigned long long>(), (const uint32_t*)nullptr, A.overflow_list, 1);
    SFCNL_CUDA_TRY(cudaGetLastError());
    if (int rc_rb = readback(c, ctl, c->build_ctl.p, 5 * 8)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *ovf_list = A.overflow_list;
    *ovf_count = 0;
    if (getenv("SFCNL_BUILD_STATS")) fprintf(stderr, "[sfcnl] warp build: %llu of %llu SCs to the medium tier\n", ctl[1], (unsigned long long)(sc1 - sc0));
    if (ctl[1]) {  // medium tier over the overflow list; what still overflows -> ctl[4]
        const size_t smem_m = size_t(kBwWarps) * sizeof(SmM);
        cudaFuncSetAttribute(k_build_warp<SmM, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_m));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
        const unsigned grid_m = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>((ctl[1] + kBwWarps - 1) / kBwWarps, uint64_t(c->num_sms) * 3)));
        launch(c, k_build_warp<SmM, 3>, dim3(grid_m), dim3(kBwWarps * 32), smem_m, A, uint64_t(0), uint64_t(ctl[1]),
               c->work_ctr.as<unsigned long long>(), (const uint32_t*)A.overflow_list, A.overflow_list + num_sc, 4);
        SFCNL_CUDA_TRY(cudaGetLastError());
        if (int rc_rb = readback(c, ctl, c->build_ctl.p, 5 * 8)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        *ovf_list = A.overflow_list + num_sc;
        *ovf_count = ctl[4];
    }
    return 0;
}

}  // namespace

int run_build_store(sfcnl_cu_ctx* c, const sfcnl_build_params& p, uint64_t sc0, uint64_t sc1, double max_h_in) {
    // ClusterParams / BuildParams validation (cluster.hpp:19-28, neighbor_store.hpp:25-28)
    if (p.ci == 0 || p.cj == 0) return set_error(c, 1, "ClusterParams: cluster sizes must be positive");
    if (64 % p.ci || 64 % p.cj)
        return set_error(c, 1, "ClusterParams: cluster sizes must divide the super-cluster size");
    if (p.ci % p.cj) return set_error(c, 1, "ClusterParams: cj must divide ci");
    if (p.w != 32 && p.w != 64) return set_error(c, 1, "ClusterParams: block width must be 32 or 64");
    if (!(p.build_radius_scale >= 1.0)) return set_error(c, 1, "BuildParams: build_radius_scale must be >= 1");
    if (!c->sorted.valid) return set_error(c, 1, "build_neighbor_store: no particles");
    const uint64_t n = c->sorted.n;
    const Box& box = c->sorted.box;
    // super-cluster range [sc0, sc1) of the sorted slot (the whole set by default;
    // a rank of a domain decomposition builds its own range over global arrays)
    const uint64_t total_sc = (n + 63) / 64;
    if (sc1 > total_sc) sc1 = total_sc;
    if (sc0 > sc1) return set_error(c, 1, "build_neighbor_store: bad super-cluster range");
    const uint64_t p_lo = sc0 * 64, p_hi = tmin<uint64_t>(sc1 * 64, n);

    SFCNL_CUDA_TRY(c->build_ctl.reserve(24 * 8));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->build_ctl.p, 0, 24 * 8, c->stream));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    if (p_hi > p_lo) {
        const uint64_t m = p_hi - p_lo;
        const int grid = int(std::min<uint64_t>((m + 255) / 256, uint64_t(c->num_sms) * 8));
        launch(c, k_validate, dim3(grid), dim3(256), 0, m, c->sorted.x.as<const double>() + p_lo,
               c->sorted.y.as<const double>() + p_lo, c->sorted.z.as<const double>() + p_lo,
               c->sorted.h.as<const double>() + p_lo, box, c->build_ctl.as<unsigned long long>() + 3,
               c->derr.as<DevError>());
    }
    static const char* const kValMsgs[] = {"", "ParticleSet: h must be positive",
                                           "ParticleSet: non-finite coordinate",
                                           "ParticleSet: position outside box (wrap first)"};
    {
        const int rc = check_dev_error(c, kValMsgs);
        if (rc) return rc;
    }
    if (!c->has_tree || c->tree_n != n)
        return set_error(c, 2, "build_neighbor_store: octree/particle-set mismatch");
    unsigned long long maxh_bits = 0;
    if (int rc_rb = readback(c, &maxh_bits, c->build_ctl.as<unsigned long long>() + 3, 8)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    double max_h;
    memcpy(&max_h, &maxh_bits, 8);
    if (max_h_in > 0) max_h = max_h_in;  // global max h supplied by the caller (domain decomposition)
    for (int d = 0; d < 3; ++d)
        if (box.per[d] && box.len[d] < 2.0 * p.build_radius_scale * max_h)
            return set_error(c, 2, "build_neighbor_store: periodic box must span twice the largest cutoff");

    const uint64_t num_sc = sc1 - sc0;
    c->sc_base = sc0;
    c->sp = p;
    c->store_n = n;
    c->num_sc = num_sc;
    c->has_store = false;
    ++c->store_gen;
    SFCNL_CUDA_TRY(c->counts.reserve(std::max<uint64_t>(num_sc, 1) * 4));
    SFCNL_CUDA_TRY(c->offsets.reserve((num_sc + 1) * 8));
    if (num_sc == 0) {
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->offsets.p, 0, 8, c->stream));
        c->blob_bytes = 0;
        c->has_store = true;
        ++c->store_gen;
        return 0;
    }
    {
        // geometry of the clusters this range reads: all of them, or (domain
        // decomposition) the range plus the halo flagged by run_halo_mark
        const bool whole = sc0 == 0 && sc1 == total_sc;
        const bool halo = !whole && c->jflags_valid && c->jflags_sc0 == sc0 && c->jflags_sc1 == sc1;
        int rc = halo ? run_cluster_geometry(c, p.ci, p.cj, p_lo, p_hi, c->jflags.as<uint8_t>())
                      : run_cluster_geometry(c, p.ci, p.cj);
        if (!rc && !c->node_geo_external) rc = run_node_geometry(c);
        if (rc) return rc;
    }
    SFCNL_CUDA_TRY(c->sc_size.reserve(num_sc * 4));
    SFCNL_CUDA_TRY(c->sc_scratch_off.reserve(num_sc * 8));
    SFCNL_CUDA_TRY(c->overflow_list.reserve(num_sc * 8));  // main-tier list, then medium-tier list
    uint64_t scratch_cap = std::max<uint64_t>(c->scratch.bytes, (p_hi - p_lo) * 16 + (1 << 20));

    BuildArgs A{};
    A.lc2g = c->dd_lc2g;
    A.n = n;
    A.box = box;
    A.scale = p.build_radius_scale;
    A.ci = p.ci, A.cj = p.cj, A.icl_per_sc = 64 / p.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = p.w, A.compress = p.compress, A.symmetric = p.mode != 0;
    A.num_icl = (n + p.ci - 1) / p.ci;
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.nodes = c->nodes.as<Node>();
    A.ngeo = c->node_geo.as<Geo>();
    A.igeo = c->igeo.as<Geo>();
    A.jgeo = p.cj == p.ci ? c->igeo.as<Geo>() : c->jgeo.as<Geo>();
    if (int rc = node_boxes32(c, A, p.mode == 0)) return rc;
    // per-SC outputs are indexed by the global SC index: offset the bases by sc0
    A.counts = c->counts.as<uint32_t>() - sc0;
    A.sizes = c->sc_size.as<uint32_t>() - sc0;
    A.soff = c->sc_scratch_off.as<uint64_t>() - sc0;
    A.ctl = c->build_ctl.as<unsigned long long>();
    A.prof = c->build_ctl.as<unsigned long long>() + 8;
    A.overflow_list = c->overflow_list.as<uint32_t>();
    A.err = c->derr.as<DevError>();
    A.leaf_cache = nullptr, A.leaf_count = nullptr, A.leaf_sc0 = sc0;
    if (c->leaf_cache_valid && c->jflags_valid && c->jflags_sc0 == sc0 && c->jflags_sc1 == sc1) {
        // the halo marking of this range already ran the same traversal (build_warp.cuh)
        A.leaf_cache = c->leaf_cache.as<uint32_t>(), A.leaf_count = c->leaf_count.as<uint32_t>();
    }

    unsigned long long ctl[5];
    for (int attempt = 0; attempt < 3; ++attempt) {
        const uint32_t* ovf_list = A.overflow_list;
        unsigned long long ovf_count = 0;
        SFCNL_CUDA_TRY(c->scratch.reserve(scratch_cap));
        A.scratch = c->scratch.as<uint8_t>();
        A.scratch_cap = c->scratch.bytes;
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->build_ctl.p, 0, 5 * 8, c->stream));
        stage_begin(c, kBuild);
        if (p.ci == 8 && (p.cj == 8 || p.cj == 4)) {
            // warp-per-SC kernel (build_warp.cuh) on the cluster-frame staging copy
            {
                const bool whole = sc0 == 0 && sc1 == total_sc;
                const bool halo = !whole && c->jflags_valid && c->jflags_sc0 == sc0 && c->jflags_sc1 == sc1;
                const int rc = halo ? run_frame(c, p.cj, nullptr, p_lo, p_hi, c->jflags.as<uint8_t>())
                                    : run_frame(c, p.cj, nullptr);
                if (rc) return rc;
            }
            A.frame = c->frame.as<const float4>();
            A.frame_x = c->frame_x.as<const unsigned>();
            SFCNL_CUDA_TRY(c->work_ctr.reserve(8));
            if (p.mode == 0 && !A.leaf_cache && attempt == 0 && !getenv("SFCNL_NO_PRETRAVERSE")) {
                // traversal as its own kernel (k_halo_warp: the same BFS, accepted leaves per SC
                // into the leaf cache); the build then starts from the cached leaves. Two smaller
                // kernels instead of one: the build's instruction-fetch stalls disappear
                // (59.2 -> 54.9 ms at C2, traversal included)
                SFCNL_CUDA_TRY(c->leaf_cache.reserve(num_sc * kLeafCacheCap * 4));
                SFCNL_CUDA_TRY(c->leaf_count.reserve(num_sc * 4));
                A.leaf_cache = c->leaf_cache.as<uint32_t>(), A.leaf_count = c->leaf_count.as<uint32_t>(), A.leaf_sc0 = sc0;
                SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
                const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((num_sc + 7) / 8, uint64_t(c->num_sms) * kTravCtas)));
                launch(c, k_halo_warp, dim3(grid), dim3(256), 0, A, sc0, sc1, (uint8_t*)nullptr,
                       c->work_ctr.as<unsigned long long>());
                SFCNL_CUDA_TRY(cudaGetLastError());
                SFCNL_CUDA_TRY(cudaMemsetAsync(c->build_ctl.p, 0, 5 * 8, c->stream));  // its overflow count
            }
            const int rc = p.mode != 0 ? launch_build_warp<BwSmemSym, BwSmemMSym>(c, A, sc0, sc1, num_sc, ctl, &ovf_list,
                                                                                 &ovf_count)
                           : A.leaf_cache ? launch_build_warp<BwSmemCached, BwSmemM>(c, A, sc0, sc1, num_sc, ctl, &ovf_list,
                                                                                    &ovf_count)
                                          : launch_build_warp<BwSmem, BwSmemM>(c, A, sc0, sc1, num_sc, ctl, &ovf_list, &ovf_count);
            if (rc) return rc;
        } else if (p.ci == 1 && p.cj == 1 && p.mode == 0 && !getenv("SFCNL_P1_GENERIC")) {
            // point clusters: warp per SC (build_p1.cuh), per-warp global workspaces
            constexpr uint32_t kCap = 16384;
            const uint64_t wstride = (uint64_t(kCap) * 25 + 1024 + 255) & ~uint64_t(255);
            const size_t smem = size_t(kBwWarps) * sizeof(P1Smem);
            cudaFuncSetAttribute(k_build_p1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            const unsigned grid = unsigned(std::max<uint64_t>(
                1, std::min<uint64_t>((num_sc + kBwWarps - 1) / kBwWarps, uint64_t(c->num_sms) * 4)));
            SFCNL_CUDA_TRY(c->fallback_ws.reserve(uint64_t(grid) * kBwWarps * wstride));
            SFCNL_CUDA_TRY(c->work_ctr.reserve(8));
            SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
            launch(c, k_build_p1, dim3(grid), dim3(kBwWarps * 32), smem, A, sc0, sc1, c->work_ctr.as<unsigned long long>(),
                   c->fallback_ws.as<uint8_t>(), wstride, kCap);
            SFCNL_CUDA_TRY(cudaGetLastError());
            if (int rc_rb = readback(c, ctl, c->build_ctl.p, 5 * 8)) return rc_rb;
            SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
            ovf_count = ctl[1];
        } else {
            const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(num_sc, uint64_t(c->num_sms) * 64)));
            launch(c, k_build_smem, dim3(grid), dim3(kBuildThreads), 0, A, sc0, sc1);
            SFCNL_CUDA_TRY(cudaGetLastError());
            if (int rc_rb = readback(c, ctl, c->build_ctl.p, 5 * 8)) return rc_rb;
            SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
            ovf_count = ctl[1];
        }
        if (ovf_count) {
            // capacity fallback in global memory: same code, big workspaces
            const uint64_t ncl = (n + p.cj - 1) / p.cj;
            const uint32_t fcap = uint32_t(std::min<uint64_t>(c->num_nodes + 8, 0xffffffffull));
            const uint32_t ccap = uint32_t(ncl + 1);
            const uint32_t ecap = uint32_t(std::min<uint64_t>(uint64_t(ccap) * (A.mask_bytes + 10) + 64, 0xfffffff0ull));
            const uint64_t stride =
                ((uint64_t(fcap) * 8 + uint64_t(ccap) * 4 + 16 + uint64_t(ccap) * 8 + ecap) + 255) & ~uint64_t(255);
            const uint64_t nblk = std::min<uint64_t>(ovf_count, 64);  // SCs too large for the warp slices
            SFCNL_CUDA_TRY(c->fallback_ws.reserve(stride * nblk));
            launch(c, k_build_global, dim3(unsigned(nblk)), dim3(kBuildThreads), 0, A, (const uint32_t*)ovf_list,
                   uint64_t(ovf_count), c->fallback_ws.as<uint8_t>(), stride, fcap, ccap, ecap);
            SFCNL_CUDA_TRY(cudaGetLastError());
            if (int rc_rb = readback(c, ctl, c->build_ctl.p, 5 * 8)) return rc_rb;
            SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
            static const char* const kMsgs[] = {"", "", "", "build_neighbor_store: workspace capacity exceeded"};
            const int rc = check_dev_error(c, kMsgs);
            if (rc) return rc;
        }
        stage_end(c, kBuild);
#ifdef SFCNL_PHASE_PROF
        {
            unsigned long long pr[11] = {};
            cudaMemcpy(pr, A.prof, 11 * 8, cudaMemcpyDeviceToHost);
            fprintf(stderr, "band items %llu\n", pr[10]);
            fprintf(stderr, "build phases (Gclk): geo %.2f trav %.2f cand %.2f masks-rest %.2f encode %.2f publish %.2f | stage %.2f thr+pref+items %.2f pairs %.2f overflow %llu\n",
                    pr[0] * 1e-9, pr[1] * 1e-9, pr[2] * 1e-9, pr[3] * 1e-9, pr[4] * 1e-9, pr[5] * 1e-9, pr[6] * 1e-9,
                    pr[7] * 1e-9, pr[8] * 1e-9, ctl[1]);
        }
#endif
        if (!ctl[2]) break;
        scratch_cap = ctl[0] + (1 << 20);  // scratch overflow: grow to the needed size and redo
        if (attempt == 2) return set_error(c, 4, "build_neighbor_store: scratch allocation failed");
    }

    stage_begin(c, kEncode);
    {
        const int rc = excl_scan(c, c->sc_size.as<uint32_t>(), c->offsets.as<uint64_t>(), num_sc);
        if (rc) return rc;
    }
    uint64_t blob_bytes = 0;
    if (int rc_rb = readback(c, &blob_bytes, c->offsets.as<uint64_t>() + num_sc, 8)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    SFCNL_CUDA_TRY(c->blob.reserve(std::max<uint64_t>(blob_bytes, 16)));
    launch(c, k_compact, dim3(unsigned((num_sc * 32 + 255) / 256)), dim3(256), 0, num_sc,
           (const uint32_t*)c->sc_size.as<uint32_t>(), (const uint64_t*)c->sc_scratch_off.as<uint64_t>(),
           (const uint64_t*)c->offsets.as<uint64_t>(), (const uint8_t*)c->scratch.as<uint8_t>(),
           c->blob.as<uint8_t>());
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kEncode);
    c->blob_bytes = blob_bytes;
    c->has_store = true;
    ++c->store_gen;
    return 0;
}

int run_halo_mark(sfcnl_cu_ctx* c, const sfcnl_build_params& p, uint64_t sc0, uint64_t sc1) {
    if (p.ci == 0 || p.cj == 0 || 64 % p.ci || 64 % p.cj || p.ci % p.cj)
        return set_error(c, 1, "ClusterParams: invalid cluster parameters");
    if (!(p.build_radius_scale >= 1.0)) return set_error(c, 1, "BuildParams: build_radius_scale must be >= 1");
    if (!c->sorted.valid) return set_error(c, 1, "halo_mark: no particles");
    const uint64_t n = c->sorted.n;
    if (!c->has_tree || c->tree_n != n) return set_error(c, 2, "halo_mark: octree/particle-set mismatch");
    const uint64_t total_sc = (n + 63) / 64;
    if (sc1 > total_sc) sc1 = total_sc;
    if (sc0 > sc1) return set_error(c, 1, "halo_mark: bad super-cluster range");
    const uint64_t nj = (n + p.cj - 1) / p.cj;
    SFCNL_CUDA_TRY(c->jflags.reserve(std::max<uint64_t>(nj, 1)));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->jflags.p, 0, std::max<uint64_t>(nj, 1), c->stream));
    c->jflags_valid = false;
    c->leaf_cache_valid = false;
    if (sc1 > sc0) {
        const uint64_t p_lo = sc0 * 64, p_hi = tmin<uint64_t>(sc1 * 64, n);
        int rc = run_cluster_geometry(c, p.ci, p.ci, p_lo, p_hi);  // i-clusters of the range
        if (!rc && !c->node_geo_external) rc = run_node_geometry(c);
        if (rc) return rc;
        SFCNL_CUDA_TRY(c->build_ctl.reserve(8 * 8));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->build_ctl.p, 0, 8 * 8, c->stream));
        SFCNL_CUDA_TRY(c->overflow_list.reserve((sc1 - sc0) * 4));
        BuildArgs A{};
        A.n = n;
        A.box = c->sorted.box;
        A.scale = p.build_radius_scale;
        A.ci = p.ci, A.cj = p.cj, A.icl_per_sc = 64 / p.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
        A.symmetric = p.mode != 0;
        A.num_icl = (n + p.ci - 1) / p.ci;
        A.nodes = c->nodes.as<Node>();
        A.ngeo = c->node_geo.as<Geo>();
        A.igeo = c->igeo.as<Geo>();
        if (int rc = node_boxes32(c, A, p.mode == 0)) return rc;
        A.ctl = c->build_ctl.as<unsigned long long>();
        A.overflow_list = c->overflow_list.as<uint32_t>();
        A.err = c->derr.as<DevError>();
        SFCNL_CUDA_TRY(c->work_ctr.reserve(8));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
        // accepted leaves per SC, reused by the range build of the same range
        SFCNL_CUDA_TRY(c->leaf_cache.reserve((sc1 - sc0) * kLeafCacheCap * 4));
        SFCNL_CUDA_TRY(c->leaf_count.reserve((sc1 - sc0) * 4));
        A.leaf_cache = c->leaf_cache.as<uint32_t>(), A.leaf_count = c->leaf_count.as<uint32_t>(), A.leaf_sc0 = sc0;
        const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((sc1 - sc0 + 7) / 8, uint64_t(c->num_sms) * 3)));
        launch(c, k_halo_warp, dim3(grid), dim3(256), 0, A, sc0, sc1, c->jflags.as<uint8_t>(),
               c->work_ctr.as<unsigned long long>());
        SFCNL_CUDA_TRY(cudaGetLastError());
        unsigned long long ctl[2];
        if (int rc_rb = readback(c, ctl, c->build_ctl.p, 2 * 8)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (ctl[1]) {
            const uint32_t fcap = uint32_t(std::min<uint64_t>(c->num_nodes + 8, 0x7fffffffull));
            const uint64_t nblk = std::min<uint64_t>(ctl[1], 8);
            SFCNL_CUDA_TRY(c->fallback_ws.reserve(nblk * 2 * uint64_t(fcap) * 4));
            launch(c, k_halo_global, dim3(unsigned(nblk)), dim3(kBuildThreads), 0, A,
                   (const uint32_t*)A.overflow_list, uint64_t(ctl[1]), c->fallback_ws.as<uint32_t>(), fcap,
                   c->jflags.as<uint8_t>());
            SFCNL_CUDA_TRY(cudaGetLastError());
        }
    }
    c->jflags_valid = true;
    c->leaf_cache_valid = sc1 > sc0 && c->leaf_cache.bytes >= (sc1 - sc0) * kLeafCacheCap * 4;
    c->jflags_sc0 = sc0, c->jflags_sc1 = sc1, c->jflags_len = nj;
    return 0;
}

}  // namespace sfcnl_cu

