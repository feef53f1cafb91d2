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
//   reduce<double>. Symmetric stores use the mirror rule (reduce.hpp:16-21) with
//   fp64 atomics for the j side (deterministic counts, values within 1e-12).
// precision 1 (k_pass_fast, ci == 8, cj in {4, 8}, gather): one CTA per SC, one
//   warp per i-cluster; lane = (i in cluster) x (j quarter). Each decoded block's
//   j particles are staged once in shared memory as float4 (x,y,z relative to the
//   SC's first particle, computed in fp64 then rounded; + mass), so the hot loop
//   is fp32 FMA work on shared memory. The cutoff decision is made in fp32 with a
//   guard band derived from the rounding-error bound of the relative coordinates;
//   pairs inside the band are decided by the exact fp64 reference predicate, so
//   neighbor_count (the pair set) is exact. Contributions accumulate in fp32 per
//   lane and are combined in fp64.
#include <algorithm>
#include <vector>

#include "ctx.hpp"

namespace sfcnl_cu {
namespace {

struct PassArgs {
    uint64_t n;
    Box box;
    uint32_t ci, cj, icl_per_sc, mask_bytes;
    int w, compress, symmetric;
    uint64_t num_sc, num_icl;
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
    double* out[4];
    uint32_t* cnt;
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
__global__ void __launch_bounds__(kExactThreads) k_pass_exact(PassArgs A) {
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    for (uint64_t sc = blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        sc_exact<K>(A, sc, st, s_idx, s_msk, &s_len);
    }
}

// One SC of the fp64 reference-order pass; threads >= 64 only take part in the
// block barriers (the fast kernel uses this for SCs it cannot handle safely).
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
                    if (A.symmetric && i > j && uint64_t(A.ci) * (j / A.ci) <= uint64_t(A.cj) * (i / A.cj)) continue;
                    double dx, dy, dz;
                    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
                    double rr = r;
                    if (A.symmetric) rr = dmul(A.qs, smax(hi, A.h[j]));
                    if (d2 > dmul(rr, rr)) continue;
                    double v[4];
                    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) {
                        coincident = true;
                        continue;
                    }
#pragma unroll
                    for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], v[o]);
                    ++cnt;
                    if (A.symmetric) {
#pragma unroll
                        for (int o = 0; o < NO; ++o) atomicAdd(A.out[o] + j, (NO == 4 && o < 3) ? -v[o] : v[o]);
                        atomicAdd(A.cnt + j, 1u);
                    }
                }
            }
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        if (active) {
            if (A.symmetric) {
#pragma unroll
                for (int o = 0; o < NO; ++o) atomicAdd(A.out[o] + i, acc[o]);
                atomicAdd(A.cnt + i, cnt);
            } else {
#pragma unroll
                for (int o = 0; o < NO; ++o) A.out[o][i] = acc[o];
                A.cnt[i] = cnt;
            }
        }
    }
}

// ---------------------------------------------------------------- fast kernel
constexpr int kFastThreads = 256;  // 8 warps = 8 i-clusters of 8
constexpr float kFar = 1.0e30f;

typedef unsigned long long f2;  // two packed fp32 lanes for the sm_100 FFMA2/FADD2/FMUL2 pipe
__device__ __forceinline__ f2 f2p(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2u(f2 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2 f2add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
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

// Rare slot: cutoff inside the guard band, or an LJ pair closer than 1.22 sigma
// (force-zero crossing / overflow range): the exact reference predicate and fp64
// kernel value, accumulated into the SC's shared fp64 side sums.
template <int K>
__device__ __noinline__ int rare_slot(const PassArgs& A, uint64_t i, uint64_t j, double r2,
                                      double* side) {
    const double xi = A.x[i], yi = A.y[i], zi = A.z[i], hi = A.h[i];
    double dx, dy, dz;
    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
    if (d2 > r2) return 0;
    double v[4];
    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) return -1;
    constexpr int NO = nout<K>();
#pragma unroll
    for (int o = 0; o < NO; ++o) atomicAdd(side + o, v[o]);
    return 1;
}

template <int K>
__global__ void __launch_bounds__(kFastThreads, 2) k_pass_fast(PassArgs A) {
    constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    constexpr int NO = nout<K>();
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ float4 s_j[64 * 8];
    __shared__ float4 s_jl[LJ ? 64 * 8 : 1];
    __shared__ double s_side[kSC][NO];
    __shared__ float s_red[8][4];
    __shared__ double s_o[3];
    __shared__ int s_len, s_unsafe;
    const unsigned tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint32_t il = lane >> 2, jq = lane & 3;
    const uint32_t cj = A.cj;
    const int i_local = int(warp * 8 + il);
    const float sig2 = float(A.sigma * A.sigma);
    const float eps24 = float(24.0 * A.eps), eps4 = float(4.0 * A.eps);
    const float close2 = 1.5f * sig2;  // (1.22 sigma)^2: LJ pairs this close go to fp64
    for (uint64_t sc = blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        const uint64_t p0 = sc * kSC;
        if (tid == 0) s_o[0] = A.x[p0], s_o[1] = A.y[p0], s_o[2] = A.z[p0];
        for (uint32_t k = tid; k < kSC * NO; k += kFastThreads) (&s_side[0][0])[k] = 0.0;
        __syncthreads();
        const double ox = s_o[0], oy = s_o[1], oz = s_o[2];
        const uint64_t i = p0 + uint64_t(i_local);
        const bool active = i < A.n;
        double hi = 1.0;
        double rx = 0, ry = 0, rz = 0;
        auto rel = [&](double v, double o, int d) {
            double r = dsub(v, o);
            if (A.box.per[d]) {
                const double L = A.box.len[d];
                if (r > 0.5 * L) r = dsub(r, L);
                else if (r < -0.5 * L) r = dadd(r, L);
            }
            return r;
        };
        if (active) {
            hi = A.h[i];
            rx = rel(A.x[i], ox, 0), ry = rel(A.y[i], oy, 1), rz = rel(A.z[i], oz, 2);
        }
        const double r = dmul(A.qs, hi);
        const double r2 = dmul(r, r);
        // Per-particle min-imaging against the SC origin is exact for every in-range
        // pair when max|rel_i| + max r < L/2 on each periodic axis; otherwise this SC
        // takes the exact path.
        {
            float ax = active ? float(fabs(rx)) : 0.f, ay = active ? float(fabs(ry)) : 0.f;
            float az = active ? float(fabs(rz)) : 0.f, ar = active ? float(r) : 0.f;
            for (int o = 16; o > 0; o >>= 1) {
                ax = fmaxf(ax, __shfl_xor_sync(0xffffffffu, ax, o));
                ay = fmaxf(ay, __shfl_xor_sync(0xffffffffu, ay, o));
                az = fmaxf(az, __shfl_xor_sync(0xffffffffu, az, o));
                ar = fmaxf(ar, __shfl_xor_sync(0xffffffffu, ar, o));
            }
            if (lane == 0) s_red[warp][0] = ax, s_red[warp][1] = ay, s_red[warp][2] = az, s_red[warp][3] = ar;
            __syncthreads();
            if (tid == 0) {
                float m[4] = {0.f, 0.f, 0.f, 0.f};
                for (int w = 0; w < 8; ++w)
                    for (int k = 0; k < 4; ++k) m[k] = fmaxf(m[k], s_red[w][k]);
                int unsafe = 0;
                for (int d = 0; d < 3; ++d)
                    if (A.box.per[d] && double(m[d]) + double(m[3]) >= 0.49 * A.box.len[d]) unsafe = 1;
                s_unsafe = unsafe;
            }
            __syncthreads();
        }
        if (s_unsafe) {
            sc_exact<K>(A, sc, st, s_idx, s_msk, &s_len);
            continue;
        }
        const float fxi = float(rx), fyi = float(ry), fzi = float(rz);
        const float lxi = float(rx - double(fxi)), lyi = float(ry - double(fyi)), lzi = float(rz - double(fzi));
        const f2 xi2 = f2p(fxi, fxi), yi2 = f2p(fyi, fyi), zi2 = f2p(fzi, fzi);
        const f2 lxi2 = f2p(lxi, lxi), lyi2 = f2p(lyi, lyi), lzi2 = f2p(lzi, lzi);
        const float ei = active ? fmaxf(fabsf(fxi), fmaxf(fabsf(fyi), fabsf(fzi))) : 0.f;
        const float inv_h = float(1.0 / hi);
        const f2 invh2 = f2p(inv_h, inv_h);
        f2 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;  // packed (slot a, slot b) partial sums
        uint32_t cnt = 0;
        bool coincident = false;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, &s_len);
            if (len < 0) break;
            // stage the block's j particles: fp64 relative -> fp32 (hi [+ lo for LJ])
            float emax = 0.f;
            for (uint32_t t = tid; t < uint32_t(len) * cj; t += kFastThreads) {
                const uint32_t e = t / cj, jj = t - e * cj;
                const uint64_t j = uint64_t(s_idx[e]) * cj + jj;
                float4 v = make_float4(kFar, kFar, kFar, 0.f);
                float4 vl = make_float4(0.f, 0.f, 0.f, 0.f);
                if (j < A.n) {
                    const double qx = rel(A.x[j], ox, 0), qy = rel(A.y[j], oy, 1), qz = rel(A.z[j], oz, 2);
                    v.x = float(qx), v.y = float(qy), v.z = float(qz);
                    v.w = (K == SFCNL_KERNEL_DENSITY) ? float(A.m[j]) : 0.f;
                    if (LJ) vl = make_float4(float(qx - double(v.x)), float(qy - double(v.y)), float(qz - double(v.z)), 0.f);
                    emax = fmaxf(emax, fmaxf(fabsf(v.x), fmaxf(fabsf(v.y), fabsf(v.z))));
                }
                s_j[e * 8 + jj] = v;
                if (LJ) s_jl[e * 8 + jj] = vl;
            }
            for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            if (lane == 0) s_red[warp][0] = emax;
            __syncthreads();
            float E = ei;
#pragma unroll
            for (int k = 0; k < 8; ++k) E = fmaxf(E, s_red[k][0]);
            // rounding-error guard band for d2 (see file header)
            const double ex = 1.1920928955078125e-07 * double(E) + 5.9604644775390625e-08 * r;
            const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
            const float lo = active ? __double2float_rd(r2 - guard) : -1.f;
            const float hi_t = active ? __double2float_ru(r2 + guard) : -1.f;
            // this warp's entries: bit `warp` of each entry mask
            unsigned long long mine = 0;
            {
                const bool b0 = lane < uint32_t(len) && ((s_msk[lane] >> warp) & 1ull);
                const bool b1 = lane + 32 < uint32_t(len) && ((s_msk[lane + 32] >> warp) & 1ull);
                mine = (unsigned long long)__ballot_sync(0xffffffffu, b0) |
                       ((unsigned long long)__ballot_sync(0xffffffffu, b1) << 32);
            }
            while (mine) {
                const int e = __ffsll(mine) - 1;
                mine &= mine - 1;
                const int jl0 = int(int64_t(s_idx[e]) * cj - int64_t(p0));
                // slots a = jq, b = jq + 4 (cj == 8); cj == 4 uses slot a only
                const float4 pa = s_j[e * 8 + jq];
                const float4 pb = cj == 8 ? s_j[e * 8 + jq + 4] : make_float4(kFar, kFar, kFar, 0.f);
                f2 dx = f2sub(xi2, f2p(pa.x, pb.x));
                f2 dy = f2sub(yi2, f2p(pa.y, pb.y));
                f2 dz = f2sub(zi2, f2p(pa.z, pb.z));
                if (LJ) {
                    const float4 la = s_jl[e * 8 + jq];
                    const float4 lb = cj == 8 ? s_jl[e * 8 + jq + 4] : make_float4(0.f, 0.f, 0.f, 0.f);
                    dx = f2add(dx, f2sub(lxi2, f2p(la.x, lb.x)));
                    dy = f2add(dy, f2sub(lyi2, f2p(la.y, lb.y)));
                    dz = f2add(dz, f2sub(lzi2, f2p(la.z, lb.z)));
                }
                const f2 d2p = f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx)));
                float d2a, d2b;
                f2u(d2p, d2a, d2b);
                const bool self_a = jl0 + int(jq) == i_local, self_b = jl0 + int(jq) + 4 == i_local;
                bool in_a = d2a < lo && !self_a, in_b = d2b < lo && !self_b;
                bool rare_a = !in_a && !(d2a > hi_t) && !self_a;
                bool rare_b = !in_b && !(d2b > hi_t) && !self_b;
                if (LJ) {
                    rare_a = rare_a || (in_a && d2a < close2);
                    rare_b = rare_b || (in_b && d2b < close2);
                    in_a = in_a && !(d2a < close2);
                    in_b = in_b && !(d2b < close2);
                }
                if (rare_a | rare_b) {
                    double* side = &s_side[i_local][0];
                    const uint64_t jb = uint64_t(s_idx[e]) * cj;
                    if (rare_a) {
                        const int rc = rare_slot<K>(A, i, jb + jq, r2, side);
                        cnt += rc > 0, coincident |= rc < 0;
                    }
                    if (rare_b) {
                        const int rc = rare_slot<K>(A, i, jb + jq + 4, r2, side);
                        cnt += rc > 0, coincident |= rc < 0;
                    }
                }
                cnt += uint32_t(in_a) + uint32_t(in_b);
                const f2 ma = f2p(in_a ? 1.f : 0.f, in_b ? 1.f : 0.f);
                if (K == SFCNL_KERNEL_DENSITY) {
                    // W(q)/sigma_i: 1 + 6q^2(q-1) for q <= 1/2, 2(1-q)^3 otherwise
                    float qa, qb;
                    asm("sqrt.approx.f32 %0, %1;" : "=f"(qa) : "f"(d2a));
                    asm("sqrt.approx.f32 %0, %1;" : "=f"(qb) : "f"(d2b));
                    const f2 q = f2mul(f2p(qa, qb), invh2);
                    const f2 q2 = f2mul(q, q);
                    const f2 wa = f2fma(f2mul(f2p(6.f, 6.f), q2), f2sub(q, f2p(1.f, 1.f)), f2p(1.f, 1.f));
                    float q0, q1;
                    f2u(q, q0, q1);
                    const f2 t = f2p(fmaxf(1.f - q0, 0.f), fmaxf(1.f - q1, 0.f));
                    const f2 wb = f2mul(f2mul(f2p(2.f, 2.f), t), f2mul(t, t));
                    float wa0, wa1, wb0, wb1;
                    f2u(wa, wa0, wa1);
                    f2u(wb, wb0, wb1);
                    const f2 w = f2p(q0 <= 0.5f ? wa0 : wb0, q1 <= 0.5f ? wa1 : wb1);
                    acc0 = f2fma(f2mul(f2p(pa.w, pb.w), ma), w, acc0);
                } else if (LJ) {
                    float ia, ib;
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ia) : "f"(d2a));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ib) : "f"(d2b));
                    const f2 inv2 = f2p(in_a ? ia : 0.f, in_b ? ib : 0.f);  // out/rare/self slots contribute 0
                    const f2 s2 = f2mul(f2p(sig2, sig2), inv2);
                    const f2 s6 = f2mul(f2mul(s2, s2), s2);
                    const f2 coef = f2mul(f2mul(f2mul(f2p(eps24, eps24), inv2), s6),
                                          f2fma(f2p(2.f, 2.f), s6, f2p(-1.f, -1.f)));
                    const f2 en = f2mul(f2mul(f2p(eps4, eps4), s6), f2sub(s6, f2p(1.f, 1.f)));
                    f2 cf = coef, ee = en;
                    if (K == SFCNL_KERNEL_LJ_COULOMB) {
                        const uint64_t jb = uint64_t(s_idx[e]) * cj;
                        const float qi = float(A.ck * A.q[i]);
                        const float qa = in_a ? qi * float(A.q[jb + jq]) : 0.f;
                        const float qb = in_b && cj == 8 ? qi * float(A.q[jb + jq + 4]) : 0.f;
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
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        __syncthreads();  // s_side complete
        // combine: slot pair, then the 4 j-quarter lanes of each i, in fp64
        double tot[4];
        const f2 accs[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            float a, b;
            f2u(accs[o], a, b);
            double v = double(a) + double(b);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            tot[o] = v;
        }
        uint32_t c = cnt;
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        if (active && jq == 0) {
            if (K == SFCNL_KERNEL_DENSITY) {
                const double sg = 8.0 / (kPi * hi * hi * hi);
                A.out[0][i] = sg * tot[0] + s_side[i_local][0];
            } else if (K == SFCNL_KERNEL_COUNT) {
                A.out[0][i] = double(c);
            } else {
#pragma unroll
                for (int o = 0; o < 4; ++o) A.out[o][i] = tot[o] + s_side[i_local][o < NO ? o : 0];
            }
            A.cnt[i] = c;
        }
    }
}

template <int K>
void launch_pass(sfcnl_cu_ctx* c, const PassArgs& A, bool fast) {
    if (fast) {
        const unsigned grid = unsigned(std::min<uint64_t>(A.num_sc, uint64_t(c->num_sms) * 8));
        launch(c, k_pass_fast<K>, dim3(grid), dim3(kFastThreads), 0, A);
    } else {
        const unsigned grid = unsigned(std::min<uint64_t>(A.num_sc, uint64_t(c->num_sms) * 32));
        launch(c, k_pass_exact<K>, dim3(grid), dim3(kExactThreads), 0, A);
    }
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
    for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(c->outs[o].reserve(std::max<uint64_t>(n, 1) * 8));
    SFCNL_CUDA_TRY(c->ncount.reserve(std::max<uint64_t>(n, 1) * 4));
    if (n == 0) return 0;
    const bool symmetric = c->sp.mode != 0;
    const bool fast = p.precision == 1 && !symmetric && c->sp.ci == 8 && (c->sp.cj == 8 || c->sp.cj == 4);
    if (symmetric || !fast) {
        for (int o = 0; o < no; ++o) SFCNL_CUDA_TRY(cudaMemsetAsync(c->outs[o].p, 0, n * 8, c->stream));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->ncount.p, 0, n * 4, c->stream));
    }
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    A.n = n;
    A.box = c->sorted.box;
    A.ci = c->sp.ci, A.cj = c->sp.cj, A.icl_per_sc = 64 / c->sp.ci, A.mask_bytes = (A.icl_per_sc + 7) / 8;
    A.w = c->sp.w, A.compress = c->sp.compress, A.symmetric = symmetric;
    A.num_sc = c->num_sc, A.num_icl = (n + A.ci - 1) / A.ci;
    A.counts = c->counts.as<uint32_t>(), A.offsets = c->offsets.as<uint64_t>(), A.blob = c->blob.as<uint8_t>();
    A.x = c->sorted.x.as<double>(), A.y = c->sorted.y.as<double>(), A.z = c->sorted.z.as<double>();
    A.h = c->sorted.h.as<double>();
    A.qs = p.query_scale, A.eps = p.epsilon, A.sigma = p.sigma, A.ck = p.coulomb_k;
    for (int o = 0; o < 4; ++o) A.out[o] = c->outs[o].as<double>();
    A.cnt = c->ncount.as<uint32_t>();
    A.err = c->derr.as<DevError>();
    stage_begin(c, kPass);
    switch (p.kernel) {
        case 0: launch_pass<0>(c, A, fast); break;
        case 1: launch_pass<1>(c, A, fast); break;
        case 2: launch_pass<2>(c, A, fast); break;
        default: launch_pass<3>(c, A, fast); break;
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

}  // namespace sfcnl_cu
