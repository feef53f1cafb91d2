// (5) Neighborhood pass: in-kernel decode of the compressed store + cluster-pair
// evaluation of the built-in kernels (SPH density, Lennard-Jones [+Coulomb], count).
//
// Replaces reduce<Real,K> (reduce.hpp:38-231): decode_entry_indices
// (neighbor_store.cpp:18-42) + codec::decode_into (nibble_codec.cpp:136-178) +
// the scalar/AVX2 entry loops (reduce.hpp:151-197, simd_avx2.cpp:125-214) +
// the kernels of builtin_kernels.hpp:12-95.
//
// Decode: one warp decodes a w-wide block of the SC's index list at a time
// (lane k owns difference k: popc of the block mask gives its info nibble, a warp
// scan of data-nibble counts gives its data nibbles, a warp scan of differences
// gives the indices). Blocks are streamed, so no per-SC capacity limit exists, and
// entries are consumed in ascending order.
//
// precision 0 (k_pass_exact): one thread per target particle i walks the SC's
//   entries in ascending order and its j-cluster in ascending j, evaluating the
//   reference expressions with round-to-nearest fp64 intrinsics. The per-i
//   summation order equals the reference's, so gather outputs are bit-equal to
//   reduce<double>. Symmetric stores: the three deterministic steps of pass_sym.cuh
//   (bit-equal to the reference's ordered j-side commit).
// precision 1 (ci == 8, cj in {4, 8}): warp-per-SC kernels with a dynamic work
//   counter -- k_pass_item (density, count: one (i-cluster, entry) item per lane,
//   cluster-frame staging, deterministic per-round reduction), k_pass_warp (LJ,
//   LJ+Coulomb: lane = (i, j quarter), hi + lo staging, fp64 close pairs),
//   k_pass_symw (symmetric stores: each stored pair evaluated once, both sides). The
//   cutoff decision is made in fp32 with a guard band derived from the rounding-error
//   bound of the staged coordinates; slots inside the band are decided by the exact
//   fp64 reference predicate, so neighbor_count (the pair set) is exact.
//   Contributions accumulate in fp32 per lane and are combined in fp64. Other
//   geometries run precision 0.
// Also here: the full Verlet list baseline and bench::cluster_overhead (pass_full.cuh).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "scan.hpp"

namespace sfcnl_cu {
namespace {

inline double __longlong_as_double_host(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

struct PassArgs {
    uint64_t n;
    Box box;
    uint32_t ci, cj, icl_per_sc, mask_bytes;
    int w, compress, symmetric;
    uint64_t sc_begin, num_sc, num_icl;  // super-clusters [sc_begin, num_sc) (global numbering)
    const uint32_t* counts;
    const uint64_t* offsets;
    const uint8_t* blob;
    const double* x;
    const double* y;
    const double* z;
    const double* h;
    const double* m;
    const double* q;
    double qs, eps, sigma, ck;
    double maxh;      // max h over the particles (symmetric fast pass: image-safety bound)
    float lj_close2;  // LJ pairs with d2 < lj_close2 * sigma^2 take the fp64 path
    float sig2f;      // float(sigma^2)
    const float4* frame;     // cluster-frame staging copy (frame.cu), density/count
    const unsigned* frame_x; // its max |offset| per axis (float bits)
    const unsigned* frame_xcl;  // per j-cluster max |offset| (float bits)
    double* out[4];
    uint32_t* cnt;
    const uint32_t* g2l;  // domain decomposition (dd.cu): decoded global cluster id -> local, or null
    const uint32_t* dec;       // the store's decoded index lists (k_decode_store), or null: decode in the pass
    const uint64_t* dec_base;  // first decoded entry of SC sc_begin + s
    DevError* err;
};

constexpr double kPi = 3.141592653589793;  // std::numbers::pi_v<double>

enum DecodeMsg { kMsgOk = 0, kMsgMaskSlice = 1, kMsgTruncMask = 2, kMsgTruncNib = 3, kMsgTrailing = 4, kMsgRawLen = 5, kMsgCoincident = 6 };

// Decodes block `bb` (elements [bb, bb+len)) of a compressed index list starting at
// byte `pos` of `data` (size bytes). Writes indices to out[0..len) (smem) and returns
// the new byte position; returns ~0 on truncation with *err_off set.
__device__ uint64_t warp_decode_block(const uint8_t* __restrict__ data, uint64_t size, uint64_t pos,
                                      uint32_t len, int w, uint64_t& running, uint32_t* out,
                                      uint64_t* err_off, int* err_msg) {
    const unsigned lane = lane_id();
    const uint32_t mbytes = uint32_t(w) / 8;
    if (pos + mbytes > size) {
        *err_off = pos;
        *err_msg = kMsgTruncMask;
        return ~0ull;
    }
    unsigned long long bm = 0;
    for (uint32_t b = 0; b < mbytes; ++b) bm |= (unsigned long long)data[pos + b] << (8 * b);
    const unsigned long long used = len == 64 ? bm : (bm & ((1ull << len) - 1ull));
    const uint32_t ninfo = __popcll(used);
    const uint64_t nib0 = (pos + mbytes) * 2;  // nibble index of the first info nibble
    const uint64_t limit = size * 2;
    if (nib0 + ninfo > limit) {
        *err_off = size;
        *err_msg = kMsgTruncNib;
        return ~0ull;
    }
    uint32_t nd[2], info[2], isset[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t k = lane + 32u * s;
        isset[s] = (k < 64 && ((used >> k) & 1ull)) ? 1u : 0u;
        nd[s] = 0, info[s] = 0;
        if (isset[s]) {
            const uint32_t at = __popcll(used & ((1ull << k) - 1ull));
            const uint64_t t = nib0 + at;
            info[s] = (data[t >> 1] >> (4 * (t & 1))) & 15u;
            nd[s] = info[s] < 8 ? info[s] + 1 : 0;
        }
    }
    const uint32_t inc0 = warp_incl_scan(nd[0]);
    const uint32_t tot0 = __shfl_sync(0xffffffffu, inc0, 31);
    const uint32_t inc1 = warp_incl_scan(nd[1]);
    const uint32_t ndata = tot0 + __shfl_sync(0xffffffffu, inc1, 31);
    if (nib0 + ninfo + ndata > limit) {
        *err_off = size;
        *err_msg = kMsgTruncNib;
        return ~0ull;
    }
    uint64_t dv[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        dv[s] = 1;
        if (isset[s]) {
            if (info[s] >= 8) {
                dv[s] = info[s] - 6;
            } else {
                uint64_t t = nib0 + ninfo + (s == 0 ? inc0 - nd[0] : tot0 + inc1 - nd[1]);
                uint64_t v = 0;
                for (uint32_t p = 0; p < nd[s]; ++p, ++t) v = (v << 4) | ((data[t >> 1] >> (4 * (t & 1))) & 15u);
                dv[s] = v;
            }
        }
    }
    // inclusive scan of differences in element order (s = 0 lanes, then s = 1 lanes)
    uint64_t a = warp_incl_scan(dv[0]);
    const uint64_t atot = __shfl_sync(0xffffffffu, a, 31);
    uint64_t b = warp_incl_scan(dv[1]) + atot;
    if (lane < len) out[lane] = uint32_t(running + a - 1);
    if (lane + 32 < len) out[lane + 32] = uint32_t(running + b - 1);
    const uint64_t btot = __shfl_sync(0xffffffffu, b, 31);
    // elements >= len contribute 1 each to the scans; subtract them from the running sum
    const uint32_t used_len = len;
    running += (w == 64 ? btot : atot) - (uint64_t(w) - used_len);
    return pos + mbytes + (ninfo + ndata + 1) / 2;
}

// Per-SC decode state shared by the pass kernels (one warp decodes).
struct ScStream {
    const uint8_t* rec;   // mask records
    const uint8_t* idata; // index data
    uint64_t ilen;
    uint32_t count;
    uint64_t pos;
    uint64_t running;
};

// Validates the SC slice (decode_entry_indices, neighbor_store.cpp:18-42). Returns
// false (and records the error) when the mask records do not fit.
__device__ __forceinline__ bool open_sc(const PassArgs& A, uint64_t sc, ScStream& s) {
    s.count = A.counts[sc];
    if (s.count == 0) return true;  // reduce.hpp:99 returns before decoding
    const uint64_t begin = A.offsets[sc], end = A.offsets[sc + 1];
    const uint64_t mb = uint64_t(s.count) * A.mask_bytes;
    if (begin + mb > end) {
        if (threadIdx.x == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgMaskSlice, begin);
        return false;
    }
    s.rec = A.blob + begin;
    s.idata = s.rec + mb;
    s.ilen = end - begin - mb;
    s.pos = 0;
    s.running = 0;
    if (!A.compress && s.ilen != uint64_t(s.count) * 4) {
        if (threadIdx.x == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgRawLen, s.ilen);
        return false;
    }
    return true;
}

// Warp 0 decodes the next block of up to w entries into idx[]/msk[]; returns the
// number of entries (0 at the end), or -1 on a decode error (recorded).
__device__ int next_block(const PassArgs& A, uint64_t sc, ScStream& s, uint32_t first,
                          uint32_t* idx, unsigned long long* msk, int* s_len) {
    __syncthreads();  // every warp is done with the previous block's idx/msk
    if (threadIdx.x < 32) {
        const uint32_t len = tmin<uint32_t>(uint32_t(A.w), s.count - first);
        int result = int(len);
        if (A.compress) {
            uint64_t off = 0;
            int msg = 0;
            const uint64_t np = warp_decode_block(s.idata, s.ilen, s.pos, len, A.w, s.running, idx, &off, &msg);
            if (np == ~0ull) {
                if (threadIdx.x == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off);
                result = -1;
            } else {
                s.pos = np;
                if (first + len == s.count && s.pos != s.ilen) {
                    if (threadIdx.x == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, s.pos);
                    result = -1;
                }
            }
        } else {
            for (uint32_t k = threadIdx.x; k < len; k += 32) {
                const uint8_t* p = s.idata + 4ull * (first + k);
                idx[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
            }
        }
        if (A.g2l && result > 0)  // same lane -> element mapping as the decode: no barrier
            for (uint32_t k = threadIdx.x; k < len; k += 32) idx[k] = A.g2l[idx[k]];
        for (uint32_t k = threadIdx.x; k < len; k += 32) {
            unsigned long long mv = 0;
            const uint8_t* r = s.rec + uint64_t(first + k) * A.mask_bytes;
            for (uint32_t b = 0; b < A.mask_bytes; ++b) mv |= (unsigned long long)r[b] << (8 * b);
            msk[k] = mv;
        }
        if (threadIdx.x == 0) *s_len = result;
    }
    __syncthreads();
    const int r = *s_len;
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- fp64 kernels
// Reference expressions with explicit rounding (builtin_kernels.hpp:12-95).
template <int K>
__device__ __forceinline__ int eval_exact(const PassArgs& A, uint64_t i, uint64_t j, double d2,
                                          double dx, double dy, double dz, double hi, double v[4]) {
    if (K == SFCNL_KERNEL_COUNT) {
        v[0] = 1.0;
    } else if (K == SFCNL_KERNEL_DENSITY) {
        const double r = __dsqrt_rn(d2);
        const double q = ddiv(r, hi);
        double w = 0.0;
        if (!(q > 1.0)) {
            const double sg = ddiv(8.0, dmul(dmul(dmul(kPi, hi), hi), hi));
            if (q <= 0.5) {
                w = dmul(sg, dadd(1.0, dmul(dmul(dmul(6.0, q), q), dsub(q, 1.0))));
            } else {
                const double t = dsub(1.0, q);
                w = dmul(dmul(dmul(dmul(sg, 2.0), t), t), t);
            }
        }
        v[0] = dmul(A.m[j], w);
    } else {
        if (d2 == 0.0) return 1;
        const double inv2 = ddiv(1.0, d2);
        const double s2 = dmul(dmul(A.sigma, A.sigma), inv2);
        const double s6 = dmul(dmul(s2, s2), s2);
        double coef = dmul(dmul(dmul(24.0, A.eps), inv2), dsub(dmul(dmul(2.0, s6), s6), s6));
        double en = dmul(dmul(4.0, A.eps), dsub(dmul(s6, s6), s6));
        if (K == SFCNL_KERNEL_LJ_COULOMB) {
            const double qq = dmul(dmul(A.ck, A.q[i]), A.q[j]);
            const double inv_r = __dsqrt_rn(inv2);
            en = dadd(en, dmul(qq, inv_r));
            coef = dadd(coef, dmul(dmul(qq, inv_r), inv2));
        }
        v[0] = dmul(coef, dx), v[1] = dmul(coef, dy), v[2] = dmul(coef, dz), v[3] = en;
    }
    return 0;
}

template <int K>
constexpr int nout() { return (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB) ? 4 : 1; }

constexpr int kExactThreads = 64;

template <int K>
__device__ __noinline__ void sc_exact(const PassArgs& A, uint64_t sc, ScStream& st, uint32_t* s_idx,
                         unsigned long long* s_msk, int* s_len);

template <int K>
__global__ void __launch_bounds__(kExactThreads) k_pass_exact(const __grid_constant__ PassArgs A) {
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        sc_exact<K>(A, sc, st, s_idx, s_msk, &s_len);
    }
}

// One SC of the fp64 reference-order pass for gather stores of any cluster shape
// (symmetric stores take pass_sym.cuh);
// threads >= 64 only take part in the block barriers.
template <int K>
__device__ __noinline__ void sc_exact(const PassArgs& A, uint64_t sc, ScStream& st, uint32_t* s_idx,
                         unsigned long long* s_msk, int* s_len) {
    constexpr int NO = nout<K>();
    const uint32_t t = threadIdx.x;
    {
        const uint64_t i = sc * kSC + t;
        const uint32_t b = t / A.ci;
        const uint64_t gi = sc * A.icl_per_sc + b;
        const bool active = t < kSC && i < A.n && gi < A.num_icl;
        double hi = 0, xi = 0, yi = 0, zi = 0;
        if (active) hi = A.h[i], xi = A.x[i], yi = A.y[i], zi = A.z[i];
        const double r = dmul(A.qs, hi);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t cnt = 0;
        bool coincident = false;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, s_len);
            if (len < 0) break;
            if (!active) continue;
            for (int e = 0; e < len; ++e) {
                if (!((s_msk[e] >> b) & 1ull)) continue;
                const uint64_t jb = uint64_t(s_idx[e]) * A.cj, je = tmin<uint64_t>(jb + A.cj, A.n);
                for (uint64_t j = jb; j < je; ++j) {
                    if (i == j) continue;
                    double dx, dy, dz;
                    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
                    if (d2 > dmul(r, r)) continue;
                    double v[4];
                    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) {
                        coincident = true;
                        continue;
                    }
#pragma unroll
                    for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], v[o]);
                    ++cnt;
                }
            }
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        if (active) {
#pragma unroll
            for (int o = 0; o < NO; ++o) A.out[o][i] = acc[o];
            A.cnt[i] = cnt;
        }
    }
}

#include "pass_fast.cuh"
#include "pass_warp.cuh"
#include "pass_item.cuh"
#include "pass_p1.cuh"
#include "pass_full.cuh"
#include "pass_sym.cuh"
#include "pass_symf.cuh"
#include "pass_x64.cuh"

// One decode per store (codec::decode_into, nibble_codec.cpp:136-178, with
// decode_entry_indices' checks, neighbor_store.cpp:18-42), shared by every pass over it:
// warp per SC, raw cluster ids (the domain decomposition's g2l map is applied by the
// passes), errors recorded exactly as the passes record them.
constexpr uint32_t kDecStage = 1024;  // bytes of an SC's index data staged in shared memory per warp
constexpr uint32_t kDecSlack = 16;    // readable bytes past the staged data (word windows)

__device__ __forceinline__ uint32_t nib_rev32(uint32_t x) {  // nibble order reversed
    x = __byte_perm(x, 0, 0x0123);
    return ((x >> 4) & 0x0F0F0F0Fu) | ((x & 0x0F0F0F0Fu) << 4);
}
// 8 bytes starting at p (shared memory, any alignment) as a little-endian word
__device__ __forceinline__ uint64_t smem_win8(const uint8_t* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = 8u * uint32_t(a & 3), w0 = w[0], w1 = w[1], w2 = w[2];
    return (uint64_t(__funnelshift_r(w1, w2, sh)) << 32) | __funnelshift_r(w0, w1, sh);
}

// warp_decode_block over the staged shared-memory copy (bytes [0, size) valid, kDecSlack
// readable beyond): a difference's nibbles come from one 8-byte window (nibble-reversed
// instead of a dependent byte loop), and the sums run in 32 bits -- the outputs are the
// low 32 bits of the same sums, the error checks and offsets are warp_decode_block's
template <int NS>  // element slots per lane: 1 for w <= 32, 2 for w = 64
__device__ __forceinline__ uint32_t warp_decode_block_s(const uint8_t* data, uint32_t size, uint32_t pos, uint32_t len,
                                                        int w, uint32_t& running, uint32_t* out, uint64_t* err_off,
                                                        int* err_msg) {
    const unsigned lane = lane_id();
    const uint32_t mbytes = uint32_t(w) / 8;
    if (pos + mbytes > size) {
        *err_off = pos;
        *err_msg = kMsgTruncMask;
        return ~0u;
    }
    const uint64_t win = smem_win8(data + pos);
    const unsigned long long bm = mbytes == 8 ? win : (win & ((1ull << (8 * mbytes)) - 1ull));
    const unsigned long long used = len == 64 ? bm : (bm & ((1ull << len) - 1ull));
    const uint32_t ninfo = __popcll(used);
    const uint32_t nib0 = (pos + mbytes) * 2, limit = size * 2;
    if (nib0 + ninfo > limit) {
        *err_off = size;
        *err_msg = kMsgTruncNib;
        return ~0u;
    }
    uint32_t nd[2] = {0, 0}, info[2] = {0, 0}, isset[2] = {0, 0};
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const uint32_t k = lane + 32u * s;
        isset[s] = ((used >> k) & 1ull) ? 1u : 0u;
        if (isset[s]) {
            const uint32_t t = nib0 + __popcll(used & ((1ull << k) - 1ull));
            info[s] = (data[t >> 1] >> (4 * (t & 1))) & 15u;
            nd[s] = info[s] < 8 ? info[s] + 1 : 0;
        }
    }
    const uint32_t inc0 = warp_incl_scan(nd[0]);
    const uint32_t tot0 = __shfl_sync(0xffffffffu, inc0, 31);
    const uint32_t inc1 = NS == 2 ? warp_incl_scan(nd[1]) : 0u;
    const uint32_t ndata = tot0 + (NS == 2 ? __shfl_sync(0xffffffffu, inc1, 31) : 0u);
    if (nib0 + ninfo + ndata > limit) {
        *err_off = size;
        *err_msg = kMsgTruncNib;
        return ~0u;
    }
    uint32_t dv[2] = {1, 1};
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        if (isset[s]) {
            if (info[s] >= 8) {
                dv[s] = info[s] - 6;
            } else {
                const uint32_t t = nib0 + ninfo + (s == 0 ? inc0 - nd[0] : tot0 + inc1 - nd[1]);
                const uint32_t seg = uint32_t(smem_win8(data + (t >> 1)) >> (4 * (t & 1)));
                dv[s] = nib_rev32(seg) >> (32 - 4 * nd[s]);
            }
        }
    }
    const uint32_t a = warp_incl_scan(dv[0]);
    const uint32_t atot = __shfl_sync(0xffffffffu, a, 31);
    if (lane < len) out[lane] = running + a - 1;
    if (NS == 2) {
        const uint32_t b = warp_incl_scan(dv[1]) + atot;
        if (lane + 32 < len) out[lane + 32] = running + b - 1;
        running += __shfl_sync(0xffffffffu, b, 31) - (uint32_t(w) - len);
    } else {
        running += atot - (uint32_t(w) - len);
    }
    return pos + mbytes + (ninfo + ndata + 1) / 2;
}
__global__ void __launch_bounds__(256) k_decode_store(const __grid_constant__ PassArgs A, uint32_t* __restrict__ dec) {
    __shared__ __align__(16) uint8_t sbuf[8][kDecStage];
    const unsigned lane = lane_id(), wp = threadIdx.x >> 5;
    const uint32_t w = uint32_t(A.w);
    // static warp-strided SCs: the decode cost per SC is nearly uniform, and one shared
    // work counter (a same-address atomic per SC) capped the kernel at ~2.3 ms for 2^20 SCs
    const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t sc = A.sc_begin + uint64_t(blockIdx.x) * (blockDim.x >> 5) + wp; sc < A.num_sc; sc += nwarps) {
        const uint32_t count = A.counts[sc];
        if (!count) continue;
        const uint64_t begin = A.offsets[sc], end = A.offsets[sc + 1];
        const uint64_t mb = uint64_t(count) * A.mask_bytes;
        if (begin + mb > end) {
            if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgMaskSlice, begin);
            continue;
        }
        const uint8_t* idata = A.blob + begin + mb;
        const uint64_t ilen = end - begin - mb;
        uint32_t* out = dec + A.dec_base[sc - A.sc_begin];
        if (!A.compress) {
            if (ilen != uint64_t(count) * 4) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgRawLen, ilen);
                continue;
            }
            for (uint32_t k = lane; k < count; k += 32) {
                const uint8_t* p = idata + 4ull * k;
                out[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
            }
            continue;
        }
        // stage the index data in one coalesced sweep (aligned words, head / tail bytes);
        // the block decodes then read shared memory instead of dependent global byte loads
        const uint8_t* src = idata;
        const bool staged = ilen + 3 + kDecSlack <= kDecStage;
        if (staged) {
            const uint64_t gs = reinterpret_cast<uint64_t>(idata), ge = gs + ilen;
            const uint64_t ws = (gs + 3) & ~3ull, we = ge & ~3ull;
            uint8_t* base = sbuf[wp] + (gs & 3);  // base[a - gs] holds the byte at address a
            if (ws < we) {
                const uint32_t* g = reinterpret_cast<const uint32_t*>(ws);
                uint32_t* d = reinterpret_cast<uint32_t*>(base + (ws - gs));
                for (uint32_t k = lane; k < uint32_t((we - ws) >> 2); k += 32) d[k] = __ldg(g + k);
                if (lane < ws - gs) base[lane] = idata[lane];
                if (lane < ge - we) base[(we - gs) + lane] = idata[(we - gs) + lane];
            } else {
                for (uint32_t k = lane; k < ilen; k += 32) base[k] = idata[k];
            }
            __syncwarp();
            src = base;
        }
        if (staged) {
            uint32_t pos = 0, running = 0;
            for (uint32_t bb = 0; bb < count; bb += w) {
                const uint32_t len = tmin<uint32_t>(w, count - bb);
                uint64_t off = 0;
                int msg = 0;
                const uint32_t np2 = w > 32 ? warp_decode_block_s<2>(src, uint32_t(ilen), pos, len, int(w), running, out + bb, &off, &msg)
                                            : warp_decode_block_s<1>(src, uint32_t(ilen), pos, len, int(w), running, out + bb, &off, &msg);
                if (np2 == ~0u) {
                    if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off);
                    break;
                }
                pos = np2;
                if (bb + len == count && pos != ilen) {
                    if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, pos);
                    break;
                }
            }
            __syncwarp();  // the staging buffer is reused by the next SC
            continue;
        }
        uint64_t pos = 0, running = 0;
        for (uint32_t bb = 0; bb < count; bb += w) {
            const uint32_t len = tmin<uint32_t>(w, count - bb);
            uint64_t off = 0;
            int msg = 0;
            const uint64_t np2 = warp_decode_block(src, ilen, pos, len, int(w), running, out + bb, &off, &msg);
            if (np2 == ~0ull) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off);
                break;
            }
            pos = np2;
            if (bb + len == count && pos != ilen) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, pos);
                break;
            }
        }
        __syncwarp();  // the staging buffer is reused by the next SC
    }
}

// The decoded lists of the current store (decoded once per store generation).
int ensure_decoded(sfcnl_cu_ctx* c, PassArgs& A) {
    A.dec = nullptr, A.dec_base = nullptr;
    if (getenv("SFCNL_NO_PREDECODE")) return 0;
    const uint64_t num_sc = A.num_sc - A.sc_begin;
    if (num_sc == 0) return 0;
    if (c->dec_gen != c->store_gen) {
        SFCNL_CUDA_TRY(c->dec_base.reserve((num_sc + 1) * 8));
        if (int rc = excl_scan(c, A.counts + A.sc_begin, c->dec_base.as<uint64_t>(), num_sc)) return rc;
        uint64_t total = 0;
        if (int rc_rb = readback(c, &total, c->dec_base.as<uint64_t>() + num_sc, 8)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        SFCNL_CUDA_TRY(c->dec_idx.reserve(std::max<uint64_t>(total, 1) * 4));
        A.dec_base = c->dec_base.as<const uint64_t>();
        const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((num_sc + 7) / 8, uint64_t(c->num_sms) * 8)));
        launch(c, k_decode_store, dim3(grid), dim3(256), 0, A, c->dec_idx.as<uint32_t>());
        SFCNL_CUDA_TRY(cudaGetLastError());
        DevError e{};
        if (int rc_rb = readback(c, &e, c->derr.p, sizeof(DevError))) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (e.key != ~0ull) {  // a malformed store: the pass decodes (and reports) it itself
            A.dec_base = nullptr;
            return 0;
        }
        c->dec_gen = c->store_gen;
    }
    A.dec = c->dec_idx.as<const uint32_t>();
    A.dec_base = c->dec_base.as<const uint64_t>();
    return 0;
}

template <int K, int CJ>
void launch_pass_warp(sfcnl_cu_ctx* c, const PassArgs& A) {
    const size_t smem = pw_smem<K>();
    cudaFuncSetAttribute(k_pass_warp<K, CJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_warp<K, CJ>, kPwWarps * 32, smem);
    const uint64_t warps = A.num_sc - A.sc_begin;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + kPwWarps - 1) / kPwWarps,
                                                                            uint64_t(c->num_sms) * std::max(per_sm, 1))));
    cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream);
    launch(c, k_pass_warp<K, CJ>, dim3(grid), dim3(kPwWarps * 32), smem, A, c->work_ctr.as<unsigned long long>());
}

template <int K, int CJ, bool NM>
void launch_pass_item_t(sfcnl_cu_ctx* c, const PassArgs& A) {
    const size_t smem = pi_smem<K>();
    cudaFuncSetAttribute(k_pass_item<K, CJ, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_item<K, CJ, NM>, kPiWarps * 32, smem);
    const uint64_t warps = A.num_sc - A.sc_begin;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + kPiWarps - 1) / kPiWarps,
                                                                            uint64_t(c->num_sms) * std::max(per_sm, 1))));
    cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream);
    launch(c, k_pass_item<K, CJ, NM>, dim3(grid), dim3(kPiWarps * 32), smem, A, c->work_ctr.as<unsigned long long>());
}

template <int K, int CJ>
void launch_pass_item(sfcnl_cu_ctx* c, const PassArgs& A) {
    // density at query scale >= 1: W(q) = 0 beyond the support, so out-of-range slots need no mask
    if (K == SFCNL_KERNEL_DENSITY && SFCNL_PI_NOMASK && A.qs >= 1.0) launch_pass_item_t<K, CJ, true>(c, A);
    else launch_pass_item_t<K, CJ, false>(c, A);
}

template <int K>
void launch_pass_p1(sfcnl_cu_ctx* c, const PassArgs& A) {
    const size_t smem = size_t(kPiWarps) * sizeof(P1pSmem);
    cudaFuncSetAttribute(k_pass_p1<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_p1<K>, kPiWarps * 32, smem);
    const uint64_t warps = A.num_sc - A.sc_begin;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + kPiWarps - 1) / kPiWarps,
                                                                            uint64_t(c->num_sms) * std::max(per_sm, 1))));
    cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream);
    launch(c, k_pass_p1<K>, dim3(grid), dim3(kPiWarps * 32), smem, A, c->work_ctr.as<unsigned long long>());
}

template <int K, int CJ>
void launch_pass_x64(sfcnl_cu_ctx* c, const PassArgs& A) {
    const size_t smem = px_smem<K>();
    cudaFuncSetAttribute(k_pass_x64<K, CJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_x64<K, CJ>, kPxWarps * 32, smem);
    const uint64_t warps = A.num_sc - A.sc_begin;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + kPxWarps - 1) / kPxWarps,
                                                                            uint64_t(c->num_sms) * std::max(per_sm, 1))));
    cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream);
    launch(c, k_pass_x64<K, CJ>, dim3(grid), dim3(kPxWarps * 32), smem, A, c->work_ctr.as<unsigned long long>());
}

template <int K>
void launch_pass(sfcnl_cu_ctx* c, const PassArgs& A, bool fast) {
    if (fast && A.ci == 1) {  // point clusters (pass_p1.cuh)
        launch_pass_p1<K>(c, A);
        return;
    }
    constexpr bool kLJ = K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB;
    if (fast && ((kLJ && !getenv("SFCNL_PASS_ITEM_LJ")) || (!kLJ && getenv("SFCNL_DENSITY_WARP")))) {  // warp-per-SC lane = (i, j-quarter) layout (pass_warp.cuh)
        if (A.cj == 8) launch_pass_warp<K, 8>(c, A);
        else launch_pass_warp<K, 4>(c, A);
    } else if (fast) {  // item-parallel layout (pass_item.cuh)
        if (A.cj == 8) launch_pass_item<K, 8>(c, A);
        else launch_pass_item<K, 4>(c, A);
    } else if (A.ci == 8 && (A.cj == 8 || A.cj == 4) && !getenv("SFCNL_PASS_EXACT_V1")) {  // fp64, pass_x64.cuh
        if (A.cj == 8) launch_pass_x64<K, 8>(c, A);
        else launch_pass_x64<K, 4>(c, A);
    } else {
        const unsigned grid = unsigned(std::min<uint64_t>(A.num_sc - A.sc_begin, uint64_t(c->num_sms) * 32));
        launch(c, k_pass_exact<K>, dim3(grid), dim3(kExactThreads), 0, A);
    }
}

// Entries per j-cluster in ascending entry order (count, scan, fill, per-cluster sort).
int sym_transpose(sfcnl_cu_ctx* c, uint64_t num_e, uint64_t ncl, const uint32_t* ejcl) {
    auto &tcnt = c->sym[5], &tstart = c->sym[6], &tlist = c->sym[7];
    SFCNL_CUDA_TRY(tcnt.reserve((ncl + 1) * 4));
    SFCNL_CUDA_TRY(tstart.reserve((ncl + 2) * 8));  // scan of ncl + 1 counts: ncl + 2 entries
    SFCNL_CUDA_TRY(tlist.reserve(std::max<uint64_t>(num_e, 1) * 4));
    const unsigned grid_e = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((num_e + 255) / 256, uint64_t(c->num_sms) * 16)));
    SFCNL_CUDA_TRY(cudaMemsetAsync(tcnt.p, 0, (ncl + 1) * 4, c->stream));
    if (num_e) launch(c, k_sym_tcount, dim3(grid_e), dim3(256), 0, num_e, ncl, ejcl, tcnt.as<uint32_t>());
    if (int rc = excl_scan(c, tcnt.as<uint32_t>(), tstart.as<uint64_t>(), ncl + 1)) return rc;
    SFCNL_CUDA_TRY(cudaMemsetAsync(tcnt.p, 0, (ncl + 1) * 4, c->stream));
    if (num_e)
        launch(c, k_sym_tfill, dim3(grid_e), dim3(256), 0, num_e, ncl, ejcl, tstart.as<const uint64_t>(), tcnt.as<uint32_t>(),
               tlist.as<uint32_t>());
    launch(c, k_sym_tsort, dim3(unsigned(std::max<uint64_t>(1, std::min<uint64_t>((ncl + 255) / 256, uint64_t(c->num_sms) * 16)))),
           dim3(256), 0, ncl, tstart.as<const uint64_t>(), tlist.as<uint32_t>());
    return 0;
}

// Global entry base per SC (exclusive scan of the counts) and the total entry count.
int sym_entry_base(sfcnl_cu_ctx* c, const PassArgs& A, uint64_t num_sc, uint64_t* num_e) {
    auto& ebase = c->sym[0];
    SFCNL_CUDA_TRY(ebase.reserve((num_sc + 1) * 8));
    if (int rc = excl_scan(c, A.counts + A.sc_begin, ebase.as<uint64_t>(), num_sc)) return rc;
    uint64_t last = 0;
    uint32_t lastc = 0;
    if (int rc_rb = readback(c, &last, ebase.as<uint64_t>() + num_sc - 1, 8)) return rc_rb;
    if (int rc_rb = readback(c, &lastc, A.counts + A.num_sc - 1, 4)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *num_e = last + lastc;
    return 0;
}

// Symmetric stores, precision 0: the three-step deterministic pass of pass_sym.cuh.
template <int K>
int launch_sym(sfcnl_cu_ctx* c, const PassArgs& A) {
    constexpr int NO = nout<K>();
    const uint64_t num_sc = A.num_sc - A.sc_begin;
    if (num_sc == 0) return 0;
    uint64_t num_e = 0;
    if (int rc = sym_entry_base(c, A, num_sc, &num_e)) return rc;
    const uint64_t ncl = (A.n + A.cj - 1) / A.cj;
    auto &ebase = c->sym[0], &jacc = c->sym[1], &jcnt = c->sym[2], &ejcl = c->sym[3], &esc = c->sym[4];
    SFCNL_CUDA_TRY(jacc.reserve(std::max<uint64_t>(num_e, 1) * NO * A.cj * 8));
    SFCNL_CUDA_TRY(jcnt.reserve(std::max<uint64_t>(num_e, 1) * A.cj * 4));
    SFCNL_CUDA_TRY(ejcl.reserve(std::max<uint64_t>(num_e, 1) * 4));
    SFCNL_CUDA_TRY(esc.reserve(std::max<uint64_t>(num_e, 1) * 4));
    const unsigned grid_sc = unsigned(std::min<uint64_t>(num_sc, uint64_t(c->num_sms) * 32));
    SFCNL_CUDA_TRY(cudaMemsetAsync(ejcl.p, 0xff, std::max<uint64_t>(num_e, 1) * 4, c->stream));
    // ebase is indexed by global SC: A.sc_begin == 0 for symmetric stores (whole range)
    launch(c, k_sym_jside<K>, dim3(grid_sc), dim3(kExactThreads), 0, A, ebase.as<const uint64_t>(), jacc.as<double>(),
           jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), esc.as<uint32_t>());
    if (int rc = sym_transpose(c, num_e, ncl, ejcl.as<const uint32_t>())) return rc;
    launch(c, k_sym_final<K>, dim3(grid_sc), dim3(kExactThreads), 0, A, jacc.as<const double>(), jcnt.as<const uint32_t>(),
           esc.as<const uint32_t>(), c->sym[6].as<const uint64_t>(), c->sym[7].as<const uint32_t>());
    return 0;
}

__global__ void k_max_h(uint64_t n, const double* __restrict__ h, unsigned long long* out) {
    double m = 0.0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x)
        m = smax(m, h[p]);
    for (int s = 16; s > 0; s >>= 1) m = smax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if (lane_id() == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));  // h > 0: bits order like values
}

// Symmetric stores, precision 1: one evaluation per stored pair (pass_symf.cuh).
template <int K>
int launch_sym_fast(sfcnl_cu_ctx* c, PassArgs A) {
    constexpr int NO = nout<K>();
    const uint64_t num_sc = A.num_sc - A.sc_begin;
    if (num_sc == 0) return 0;
    uint64_t num_e = 0;
    if (int rc = sym_entry_base(c, A, num_sc, &num_e)) return rc;
    const uint64_t ncl = (A.n + A.cj - 1) / A.cj;
    {
        SFCNL_CUDA_TRY(c->small_host_dev.reserve(16));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->small_host_dev.p, 0, 8, c->stream));
        launch(c, k_max_h, dim3(unsigned(std::min<uint64_t>((A.n + 255) / 256, uint64_t(c->num_sms) * 8))), dim3(256), 0, A.n,
               A.h, c->small_host_dev.as<unsigned long long>());
        unsigned long long bits = 0;
        if (int rc_rb = readback(c, &bits, c->small_host_dev.p, 8)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        A.maxh = __longlong_as_double_host(bits);
    }
    constexpr int NE = PsSmem<K>::NE;
    auto &ebase = c->sym[0], &jacc = c->sym[1], &jcnt = c->sym[2], &ejcl = c->sym[3];
    SFCNL_CUDA_TRY(jacc.reserve(std::max<uint64_t>(num_e, 1) * NE * A.cj * 4));
    SFCNL_CUDA_TRY(c->sym_aux.reserve(std::max<uint64_t>(A.n, 1) * 8 + 8));
    double* aux = c->sym_aux.as<double>();
    SFCNL_CUDA_TRY(c->sym_spec.reserve(std::max<uint64_t>(A.n, 1) * NO * 8));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->sym_spec.p, 0, A.n * NO * 8, c->stream));
    double* jspec = c->sym_spec.as<double>();
    SFCNL_CUDA_TRY(jcnt.reserve(std::max<uint64_t>(num_e, 1) * A.cj * 4));
    SFCNL_CUDA_TRY(ejcl.reserve(std::max<uint64_t>(num_e, 1) * 4));
    SFCNL_CUDA_TRY(cudaMemsetAsync(ejcl.p, 0xff, std::max<uint64_t>(num_e, 1) * 4, c->stream));
    const size_t smem = ps_smem<K>();
    auto kern = A.cj == 8 ? k_pass_symw<K, 8> : k_pass_symw<K, 4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPwWarps * 32, smem);
    const unsigned grid = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>((num_sc + kPwWarps - 1) / kPwWarps, uint64_t(c->num_sms) * std::max(per_sm, 1))));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
    SFCNL_CUDA_TRY(c->sym[8].reserve(uint64_t(grid) * kPwWarps * kSqCap * 4));
    launch(c, kern, dim3(grid), dim3(kPwWarps * 32), smem, A, c->work_ctr.as<unsigned long long>(),
           ebase.as<const uint64_t>(), jacc.as<float>(), jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), c->sym[8].as<uint32_t>(), aux, jspec);
    if (int rc = sym_transpose(c, num_e, ncl, ejcl.as<const uint32_t>())) return rc;
    launch(c, k_sym_fgather<K>, dim3(unsigned(std::min<uint64_t>((A.n + 255) / 256, uint64_t(c->num_sms) * 16))), dim3(256), 0,
           A.n, uint32_t(A.cj), jacc.as<const float>(), jcnt.as<const uint32_t>(), c->sym[6].as<const uint64_t>(),
           c->sym[7].as<const uint32_t>(), A.out[0], A.out[1], A.out[2], A.out[3], A.cnt, aux, (const double*)jspec);
    if (K == SFCNL_KERNEL_DENSITY) {  // particles whose error bound exceeds the bar: the whole pass in fp64
        unsigned long long* flagged = reinterpret_cast<unsigned long long*>(aux + A.n);
        SFCNL_CUDA_TRY(cudaMemsetAsync(flagged, 0, 8, c->stream));
        launch(c, k_sym_check, dim3(unsigned(std::min<uint64_t>((A.n + 255) / 256, uint64_t(c->num_sms) * 16))), dim3(256), 0,
               A.n, A.qs, (const double*)A.out[0], (const double*)aux, flagged);
        unsigned long long nf = 0;
        if (int rc_rb = readback(c, &nf, flagged, 8)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        c->last_redo = nf;
        if (nf) return launch_sym<K>(c, A);
    }
    return 0;
}

}  // namespace

int run_reduce(sfcnl_cu_ctx* c, const sfcnl_pass_params& p) {
    if (!c->sorted.valid) return set_error(c, 1, "reduce: no particles");
    if (!c->has_store) return set_error(c, 1, "reduce: no neighbor store");
    const uint64_t n = c->sorted.n;
    if (c->store_n != n) return set_error(c, 1, "reduce: store/particle-set size mismatch");
    if (!(p.query_scale >= 0)) return set_error(c, 1, "PassConfig: query_scale must be >= 0");
    if (p.query_scale > c->sp.build_radius_scale)
        return set_error(c, 1, "reduce: query_scale exceeds the store's build radius scale");
    if (p.kernel < 0 || p.kernel > 3) return set_error(c, 1, "reduce: unknown kernel");
    PassArgs A{};
    if (p.kernel == SFCNL_KERNEL_DENSITY) {
        auto* f = c->sorted.find("m");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: m");
        A.m = f->data.as<double>();
    }
    if (p.kernel == SFCNL_KERNEL_LJ_COULOMB) {
        auto* f = c->sorted.find("q");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: q");
        A.q = f->data.as<double>();
    }
    const int no = p.kernel >= 2 ? 4 : 1;
    // A range store (sc_base > 0 or a partial range) covers particles
    // [sc_base*64, sc_base*64 + nout); outputs are indexed locally.
    const uint64_t nout = pass_out_count(c);
    const uint64_t p0 = c->sc_base * 64;
    for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(c->outs[o].reserve(std::max<uint64_t>(nout, 1) * 8));
    SFCNL_CUDA_TRY(c->ncount.reserve(std::max<uint64_t>(nout, 1) * 4));
    if (nout == 0) return 0;
    const bool symmetric = c->sp.mode != 0;
    if (symmetric && (c->sc_base != 0 || nout != n))
        return set_error(c, 1, "reduce: symmetric stores cannot be restricted to a super-cluster range");
    const bool fast = p.precision == 1 && !symmetric &&
                      ((c->sp.ci == 8 && (c->sp.cj == 8 || c->sp.cj == 4)) || (c->sp.ci == 1 && c->sp.cj == 1));
    if (symmetric || !fast) {
        for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(cudaMemsetAsync(c->outs[o].p, 0, nout * 8, c->stream));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->ncount.p, 0, nout * 4, c->stream));
    }
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    SFCNL_CUDA_TRY(c->work_ctr.reserve(8));
    if (fast && c->sp.ci == 8 && (p.kernel == SFCNL_KERNEL_DENSITY || p.kernel == SFCNL_KERNEL_COUNT)) {
        // staging copy for the item pass: the store's range (+ its halo clusters)
        const uint64_t sc0 = c->sc_base, sc1 = c->sc_base + c->num_sc;
        const bool whole = sc0 == 0 && sc1 == (n + 63) / 64;
        const bool halo = !whole && c->jflags_valid && c->jflags_sc0 == sc0 && c->jflags_sc1 == sc1;
        const int rc = halo ? run_frame(c, c->sp.cj, A.m, sc0 * 64, sc1 * 64, c->jflags.as<uint8_t>())
                            : run_frame(c, c->sp.cj, A.m);
        if (rc) return rc;
        A.frame = c->frame.as<const float4>();
        A.frame_x = c->frame_x.as<const unsigned>();
        A.frame_xcl = c->frame_xcl.as<const unsigned>();
    }
    A.n = n;
    A.box = c->sorted.box;
    A.ci = c->sp.ci, A.cj = c->sp.cj, A.icl_per_sc = 64 / c->sp.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = c->sp.w, A.compress = c->sp.compress, A.symmetric = symmetric;
    A.sc_begin = c->sc_base, A.num_sc = c->sc_base + c->num_sc, A.num_icl = (n + A.ci - 1) / A.ci;
    // store arrays are local to the range: shift them so kernels index by global SC
    A.counts = c->counts.as<uint32_t>() - c->sc_base, A.offsets = c->offsets.as<uint64_t>() - c->sc_base;
    A.blob = c->blob.as<uint8_t>();
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.qs = p.query_scale, A.eps = p.epsilon, A.sigma = p.sigma, A.ck = p.coulomb_k;
    A.lj_close2 = kLjClose2;
    A.sig2f = float(p.sigma * p.sigma);
    if (const char* e = getenv("SFCNL_LJ_CLOSE2")) A.lj_close2 = float(atof(e));
    for (int o = 0; o < 4; ++o) A.out[o] = c->outs[o].as<double>() - p0;
    A.cnt = c->ncount.as<uint32_t>() - p0;
    A.err = c->derr.as<DevError>();
    A.g2l = c->dd_g2l;
    stage_begin(c, kPass);
    if (!symmetric && A.ci == 8 && (A.cj == 8 || A.cj == 4))
        if (int rc = ensure_decoded(c, A)) return rc;
    if (symmetric) {
        const bool sym_fast = p.precision == 1 && c->sp.ci == 8 && (c->sp.cj == 8 || c->sp.cj == 4) &&
                              !getenv("SFCNL_SYM_EXACT");
        int rc = 0;
        switch (p.kernel) {
            case 0: rc = sym_fast ? launch_sym_fast<0>(c, A) : launch_sym<0>(c, A); break;
            case 1: rc = sym_fast ? launch_sym_fast<1>(c, A) : launch_sym<1>(c, A); break;
            case 2: rc = sym_fast ? launch_sym_fast<2>(c, A) : launch_sym<2>(c, A); break;
            default: rc = sym_fast ? launch_sym_fast<3>(c, A) : launch_sym<3>(c, A); break;
        }
        if (rc) return rc;
    } else {
        switch (p.kernel) {
            case 0: launch_pass<0>(c, A, fast); break;
            case 1: launch_pass<1>(c, A, fast); break;
            case 2: launch_pass<2>(c, A, fast); break;
            default: launch_pass<3>(c, A, fast); break;
        }
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kPass);
    static const char* const kMsgs[] = {"",
                                        "blob slice too short for bitmasks",
                                        "truncated bitmask",
                                        "truncated nibble stream",
                                        "trailing bytes in index blob",
                                        "raw index blob length mismatch",
                                        "reduce: coincident particles"};
    return check_dev_error(c, kMsgs);
}

// ------------------------------------------------------------ full Verlet list (f3)
int run_build_full_list(sfcnl_cu_ctx* c, double build_scale) {
    if (!c->sorted.valid) return set_error(c, 1, "build_full_list: no particles");
    if (!c->has_store) return set_error(c, 1, "build_full_list: no neighbor store");
    const uint64_t n = c->sorted.n;
    if (c->store_n != n) return set_error(c, 1, "build_full_list: store/particle-set size mismatch");
    if (c->sp.mode != 0) return set_error(c, 1, "build_full_list: the store must be a gather store");
    if (c->sc_base != 0 || c->num_sc != (n + 63) / 64)
        return set_error(c, 1, "build_full_list: the store must cover every super-cluster");
    if (!(build_scale >= 0)) return set_error(c, 1, "build_full_list: build_scale must be >= 0");
    if (build_scale > c->sp.build_radius_scale)
        return set_error(c, 1, "build_full_list: build_scale exceeds the store's build radius scale");
    if (n >= (1ull << 32)) return set_error(c, 1, "build_full_list: more than 2^32 particles");
    PassArgs A{};
    A.n = n;
    A.box = c->sorted.box;
    A.ci = c->sp.ci, A.cj = c->sp.cj, A.icl_per_sc = 64 / c->sp.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = c->sp.w, A.compress = c->sp.compress;
    A.sc_begin = 0, A.num_sc = c->num_sc, A.num_icl = (n + A.ci - 1) / A.ci;
    A.counts = c->counts.as<uint32_t>(), A.offsets = c->offsets.as<uint64_t>(), A.blob = c->blob.as<uint8_t>();
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.qs = build_scale;
    A.err = c->derr.as<DevError>();
    SFCNL_CUDA_TRY(c->full_cnt.reserve((n + 1) * 4));
    SFCNL_CUDA_TRY(c->full_off.reserve((n + 2) * 8));  // scan of n + 1 counts: n + 2 entries
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->full_cnt.p, 0, (n + 1) * 4, c->stream));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    c->has_full = false;
    stage_begin(c, kPass);
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(A.num_sc, uint64_t(c->num_sms) * 32)));
    if (A.num_sc)
        launch(c, k_full_list<false>, dim3(grid), dim3(kExactThreads), 0, A, c->full_cnt.as<uint32_t>(),
               (const uint64_t*)nullptr, (uint32_t*)nullptr);
    if (int rc = excl_scan(c, c->full_cnt.as<uint32_t>(), c->full_off.as<uint64_t>(), n + 1)) return rc;
    uint64_t pairs = 0;
    if (int rc_rb = readback(c, &pairs, c->full_off.as<uint64_t>() + n, 8)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    SFCNL_CUDA_TRY(c->full_nbr.reserve(std::max<uint64_t>(pairs, 1) * 4));
    if (A.num_sc)
        launch(c, k_full_list<true>, dim3(grid), dim3(kExactThreads), 0, A, (uint32_t*)nullptr,
               c->full_off.as<const uint64_t>(), c->full_nbr.as<uint32_t>());
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kPass);
    static const char* const kMsgs[] = {"",
                                        "blob slice too short for bitmasks",
                                        "truncated bitmask",
                                        "truncated nibble stream",
                                        "trailing bytes in index blob",
                                        "raw index blob length mismatch",
                                        ""};
    if (int rc = check_dev_error(c, kMsgs)) return rc;
    c->full_n = n, c->full_pairs = pairs, c->full_scale = build_scale, c->full_mode = 0;
    c->has_full = true;
    return 0;
}

int run_reduce_full(sfcnl_cu_ctx* c, const sfcnl_pass_params& p) {
    if (!c->sorted.valid) return set_error(c, 1, "reduce_full: no particles");
    if (!c->has_full) return set_error(c, 1, "reduce_full: no full list");
    const uint64_t n = c->sorted.n;
    if (c->full_n != n) return set_error(c, 1, "reduce_full: list/particle-set mismatch");
    if (!(p.query_scale >= 0)) return set_error(c, 1, "PassConfig: query_scale must be >= 0");
    if (p.query_scale > c->full_scale) return set_error(c, 1, "reduce_full: query_scale exceeds the list's build scale");
    if (p.kernel < 0 || p.kernel > 3) return set_error(c, 1, "reduce_full: unknown kernel");
    PassArgs A{};
    if (p.kernel == SFCNL_KERNEL_DENSITY) {
        auto* f = c->sorted.find("m");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: m");
        A.m = f->data.as<double>();
    }
    if (p.kernel == SFCNL_KERNEL_LJ_COULOMB) {
        auto* f = c->sorted.find("q");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: q");
        A.q = f->data.as<double>();
    }
    const int no = p.kernel >= 2 ? 4 : 1;
    for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(c->outs[o].reserve(std::max<uint64_t>(n, 1) * 8));
    SFCNL_CUDA_TRY(c->ncount.reserve(std::max<uint64_t>(n, 1) * 4));
    if (n == 0) return 0;
    A.n = n;
    A.box = c->sorted.box;
    A.symmetric = c->full_mode != 0;
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.qs = p.query_scale, A.eps = p.epsilon, A.sigma = p.sigma, A.ck = p.coulomb_k;
    for (int o = 0; o < 4; ++o) A.out[o] = c->outs[o].as<double>();
    A.cnt = c->ncount.as<uint32_t>();
    A.err = c->derr.as<DevError>();
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    const uint64_t* off = c->full_off.as<const uint64_t>();
    const uint32_t* nb = c->full_nbr.as<const uint32_t>();
    stage_begin(c, kPass);
    if (p.precision == 1) {
        const unsigned grid = unsigned(std::min<uint64_t>((n + 7) / 8, uint64_t(c->num_sms) * 64));
        switch (p.kernel) {
            case 0: launch(c, k_reduce_full_warp<0>, dim3(grid), dim3(256), 0, A, off, nb); break;
            case 1: launch(c, k_reduce_full_warp<1>, dim3(grid), dim3(256), 0, A, off, nb); break;
            case 2: launch(c, k_reduce_full_warp<2>, dim3(grid), dim3(256), 0, A, off, nb); break;
            default: launch(c, k_reduce_full_warp<3>, dim3(grid), dim3(256), 0, A, off, nb); break;
        }
    } else {
        const unsigned grid = unsigned(std::min<uint64_t>((n + 127) / 128, uint64_t(c->num_sms) * 16));
        switch (p.kernel) {
            case 0: launch(c, k_reduce_full_exact<0>, dim3(grid), dim3(128), 0, A, off, nb); break;
            case 1: launch(c, k_reduce_full_exact<1>, dim3(grid), dim3(128), 0, A, off, nb); break;
            case 2: launch(c, k_reduce_full_exact<2>, dim3(grid), dim3(128), 0, A, off, nb); break;
            default: launch(c, k_reduce_full_exact<3>, dim3(grid), dim3(128), 0, A, off, nb); break;
        }
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kPass);
    static const char* const kMsgs[] = {"", "", "", "", "", "", "reduce_full: coincident particles"};
    return check_dev_error(c, kMsgs);
}

int run_cluster_slots(sfcnl_cu_ctx* c, uint64_t* slots) {
    if (!c->has_store) return set_error(c, 1, "cluster_overhead: no neighbor store");
    if (c->sp.mode != 0) return set_error(c, 1, "cluster_overhead: requires a gather-mode store");
    const uint64_t n = c->store_n;
    PassArgs A{};
    A.n = n;
    A.ci = c->sp.ci, A.cj = c->sp.cj, A.icl_per_sc = 64 / c->sp.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = c->sp.w, A.compress = c->sp.compress;
    A.sc_begin = c->sc_base, A.num_sc = c->sc_base + c->num_sc, A.num_icl = (n + A.ci - 1) / A.ci;
    A.counts = c->counts.as<uint32_t>() - c->sc_base, A.offsets = c->offsets.as<uint64_t>() - c->sc_base;
    A.blob = c->blob.as<uint8_t>();
    A.err = c->derr.as<DevError>();
    SFCNL_CUDA_TRY(c->work_ctr.reserve(8));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->work_ctr.p, 0, 8, c->stream));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    if (c->num_sc) {
        const unsigned grid = unsigned(std::min<uint64_t>(c->num_sc, uint64_t(c->num_sms) * 32));
        launch(c, k_cluster_slots, dim3(grid), dim3(kExactThreads), 0, A, c->work_ctr.as<unsigned long long>());
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    static const char* const kMsgs[] = {"",
                                        "blob slice too short for bitmasks",
                                        "truncated bitmask",
                                        "truncated nibble stream",
                                        "trailing bytes in index blob",
                                        "raw index blob length mismatch",
                                        ""};
    if (int rc = check_dev_error(c, kMsgs)) return rc;
    if (int rc_rb = readback(c, slots, c->work_ctr.p, 8)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return 0;
}

// ------------------------------------------------ symmetric stores under domain decomposition
// The reference order (pass_sym.cuh) folds, per particle, the j-side accumulators of the
// entries whose j-cluster holds it in GLOBAL entry order around its own i side. With the
// SCs split over ranks, rank r computes the accumulators of its own entries
// (sym_range_entries); entries whose j-cluster another rank owns are shipped there
// (always a later rank: the half-list rule puts j at or after the entry's i-cluster);
// the owner prepends what it receives (earlier ranks, rank order = global entry order)
// to its own entries and runs the ordered fold for its particles (sym_range_final).
namespace {
int sym_range_args(sfcnl_cu_ctx* c, const sfcnl_pass_params& p, PassArgs& A, const char* who) {
    if (!c->sorted.valid) return set_error(c, 1, std::string(who) + ": no particles");
    if (!c->has_store) return set_error(c, 1, std::string(who) + ": no neighbor store");
    if (c->sp.mode == 0) return set_error(c, 1, std::string(who) + ": the store must be symmetric");
    const uint64_t n = c->sorted.n;
    if (c->store_n != n) return set_error(c, 1, "reduce: store/particle-set size mismatch");
    if (!(p.query_scale >= 0)) return set_error(c, 1, "PassConfig: query_scale must be >= 0");
    if (p.query_scale > c->sp.build_radius_scale)
        return set_error(c, 1, "reduce: query_scale exceeds the store's build radius scale");
    if (p.kernel < 0 || p.kernel > 3) return set_error(c, 1, "reduce: unknown kernel");
    A = PassArgs{};
    if (p.kernel == SFCNL_KERNEL_DENSITY) {
        auto* f = c->sorted.find("m");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: m");
        A.m = f->data.as<double>();
    }
    if (p.kernel == SFCNL_KERNEL_LJ_COULOMB) {
        auto* f = c->sorted.find("q");
        if (!f) return set_error(c, 1, "ParticleSet: no such field: q");
        A.q = f->data.as<double>();
    }
    A.n = n;
    A.box = c->sorted.box;
    A.ci = c->sp.ci, A.cj = c->sp.cj, A.icl_per_sc = 64 / c->sp.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = c->sp.w, A.compress = c->sp.compress, A.symmetric = 1;
    A.sc_begin = c->sc_base, A.num_sc = c->sc_base + c->num_sc, A.num_icl = (n + A.ci - 1) / A.ci;
    A.counts = c->counts.as<uint32_t>() - c->sc_base, A.offsets = c->offsets.as<uint64_t>() - c->sc_base;
    A.blob = c->blob.as<uint8_t>();
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.qs = p.query_scale, A.eps = p.epsilon, A.sigma = p.sigma, A.ck = p.coulomb_k;
    A.err = c->derr.as<DevError>();
    return 0;
}
}  // namespace

int run_sym_range_entries(sfcnl_cu_ctx* c, const sfcnl_pass_params& p, uint64_t* num_e) {
    PassArgs A{};
    if (int rc = sym_range_args(c, p, A, "sym_range_entries")) return rc;
    const int no = p.kernel >= 2 ? 4 : 1;
    uint64_t ne = 0;
    if (c->num_sc) {
        auto& ebase = c->sym[0];
        SFCNL_CUDA_TRY(ebase.reserve((c->num_sc + 1) * 8));
        if (int rc = excl_scan(c, c->counts.as<uint32_t>(), ebase.as<uint64_t>(), c->num_sc)) return rc;
        uint64_t last = 0;
        uint32_t lastc = 0;
        if (int rc_rb = readback(c, &last, ebase.as<uint64_t>() + c->num_sc - 1, 8)) return rc_rb;
        if (int rc_rb = readback(c, &lastc, c->counts.as<uint32_t>() + c->num_sc - 1, 4)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        ne = last + lastc;
    }
    auto &jacc = c->sym[1], &jcnt = c->sym[2], &ejcl = c->sym[3], &esc = c->sym[4];
    SFCNL_CUDA_TRY(jacc.reserve(std::max<uint64_t>(ne, 1) * no * A.cj * 8));
    SFCNL_CUDA_TRY(jcnt.reserve(std::max<uint64_t>(ne, 1) * A.cj * 4));
    SFCNL_CUDA_TRY(ejcl.reserve(std::max<uint64_t>(ne, 1) * 4));
    SFCNL_CUDA_TRY(esc.reserve(std::max<uint64_t>(ne, 1) * 4));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    SFCNL_CUDA_TRY(cudaMemsetAsync(ejcl.p, 0xff, std::max<uint64_t>(ne, 1) * 4, c->stream));
    if (c->num_sc) {
        const unsigned grid = unsigned(std::min<uint64_t>(c->num_sc, uint64_t(c->num_sms) * 32));
        const uint64_t* eb = c->sym[0].as<const uint64_t>() - c->sc_base;  // indexed by global SC
        switch (p.kernel) {
            case 0: launch(c, k_sym_jside<0>, dim3(grid), dim3(kExactThreads), 0, A, eb, jacc.as<double>(), jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), esc.as<uint32_t>()); break;
            case 1: launch(c, k_sym_jside<1>, dim3(grid), dim3(kExactThreads), 0, A, eb, jacc.as<double>(), jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), esc.as<uint32_t>()); break;
            case 2: launch(c, k_sym_jside<2>, dim3(grid), dim3(kExactThreads), 0, A, eb, jacc.as<double>(), jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), esc.as<uint32_t>()); break;
            default: launch(c, k_sym_jside<3>, dim3(grid), dim3(kExactThreads), 0, A, eb, jacc.as<double>(), jcnt.as<uint32_t>(), ejcl.as<uint32_t>(), esc.as<uint32_t>()); break;
        }
        SFCNL_CUDA_TRY(cudaGetLastError());
    }
    c->sym_e_local = ne;
    c->sym_e_kernel = p.kernel;
    static const char* const kMsgs[] = {"", "blob slice too short for bitmasks", "truncated bitmask", "truncated nibble stream",
                                        "trailing bytes in index blob", "raw index blob length mismatch", ""};
    if (int rc = check_dev_error(c, kMsgs)) return rc;
    *num_e = ne;
    return 0;
}

int run_sym_range_final(sfcnl_cu_ctx* c, const sfcnl_pass_params& p, uint64_t nr, const double* rjacc,
                        const uint32_t* rjcnt, const uint32_t* rejcl, const uint32_t* resc) {
    PassArgs A{};
    if (int rc = sym_range_args(c, p, A, "sym_range_final")) return rc;
    if (c->sym_e_kernel != p.kernel) return set_error(c, 1, "sym_range_final: run sym_range_entries for this kernel first");
    const int no = p.kernel >= 2 ? 4 : 1;
    const uint64_t cj = A.cj, nl = c->sym_e_local, nt = nr + nl;
    auto &cjacc = c->symc[0], &cjcnt = c->symc[1], &cejcl = c->symc[2], &cesc = c->symc[3];
    SFCNL_CUDA_TRY(cjacc.reserve(std::max<uint64_t>(nt, 1) * no * cj * 8));
    SFCNL_CUDA_TRY(cjcnt.reserve(std::max<uint64_t>(nt, 1) * cj * 4));
    SFCNL_CUDA_TRY(cejcl.reserve(std::max<uint64_t>(nt, 1) * 4));
    SFCNL_CUDA_TRY(cesc.reserve(std::max<uint64_t>(nt, 1) * 4));
    auto cp = [&](void* dst, const void* src, size_t bytes) -> int {
        if (bytes) SFCNL_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
        return 0;
    };
    // remote entries first (earlier ranks, in rank order), then the local ones
    if (int rc = cp(cjacc.p, rjacc, nr * no * cj * 8)) return rc;
    if (int rc = cp(cjcnt.p, rjcnt, nr * cj * 4)) return rc;
    if (int rc = cp(cejcl.p, rejcl, nr * 4)) return rc;
    if (int rc = cp(cesc.p, resc, nr * 4)) return rc;
    if (int rc = cp(cjacc.as<double>() + nr * no * cj, c->sym[1].p, nl * no * cj * 8)) return rc;
    if (int rc = cp(cjcnt.as<uint32_t>() + nr * cj, c->sym[2].p, nl * cj * 4)) return rc;
    if (int rc = cp(cejcl.as<uint32_t>() + nr, c->sym[3].p, nl * 4)) return rc;
    if (int rc = cp(cesc.as<uint32_t>() + nr, c->sym[4].p, nl * 4)) return rc;
    const uint64_t ncl = (A.n + cj - 1) / cj;
    if (int rc = sym_transpose(c, nt, ncl, cejcl.as<const uint32_t>())) return rc;
    const uint64_t nout = pass_out_count(c), p0 = c->sc_base * 64;
    for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(c->outs[o].reserve(std::max<uint64_t>(nout, 1) * 8));
    SFCNL_CUDA_TRY(c->ncount.reserve(std::max<uint64_t>(nout, 1) * 4));
    for (int o = 0; o < 4; ++o) A.out[o] = c->outs[o].as<double>() - p0;
    A.cnt = c->ncount.as<uint32_t>() - p0;
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    if (c->num_sc) {
        const unsigned grid = unsigned(std::min<uint64_t>(c->num_sc, uint64_t(c->num_sms) * 32));
        const double* ja = cjacc.as<const double>();
        const uint32_t *jc = cjcnt.as<const uint32_t>(), *es = cesc.as<const uint32_t>();
        const uint64_t* ts = c->sym[6].as<const uint64_t>();
        const uint32_t* tl = c->sym[7].as<const uint32_t>();
        switch (p.kernel) {
            case 0: launch(c, k_sym_final<0>, dim3(grid), dim3(kExactThreads), 0, A, ja, jc, es, ts, tl); break;
            case 1: launch(c, k_sym_final<1>, dim3(grid), dim3(kExactThreads), 0, A, ja, jc, es, ts, tl); break;
            case 2: launch(c, k_sym_final<2>, dim3(grid), dim3(kExactThreads), 0, A, ja, jc, es, ts, tl); break;
            default: launch(c, k_sym_final<3>, dim3(grid), dim3(kExactThreads), 0, A, ja, jc, es, ts, tl); break;
        }
        SFCNL_CUDA_TRY(cudaGetLastError());
    }
    static const char* const kMsgs[] = {"", "blob slice too short for bitmasks", "truncated bitmask", "truncated nibble stream",
                                        "trailing bytes in index blob", "raw index blob length mismatch",
                                        "reduce: coincident particles"};
    return check_dev_error(c, kMsgs);
}

}  // namespace sfcnl_cu
