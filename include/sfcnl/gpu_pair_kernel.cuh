// B200 drop-in: user pair kernels on the GPU (CUDA translation units only).
//
// reduce<Real, K> with a kernel that is not built in (make_pair_kernel /
// BasicPairKernel, pair_kernel.hpp:60-91, or any type with the same members)
// instantiates this generic device pass in the caller's CUDA translation unit: the
// reference's scalar loop (reduce.hpp:151-197) and postamble (reduce.hpp:222-229)
// restated as a kernel over the device state of the process's B200 context (the
// sorted particle set, its input fields and the store, uploaded through the C-ABI,
// include/sfcnl_cu.h section (5a)).
//
// One CTA per super-cluster, one thread per target i (64): thread 0 decodes the SC's
// index list one codec block at a time into shared memory (codec::decode_into,
// nibble_codec.cpp:136-178, with decode_entry_indices' checks, neighbor_store.cpp:
// 18-42); every thread walks the entries in ascending order and its j-cluster in
// ascending j, exactly like the reference, so each output is reduced in the same
// order. The pair geometry (min-image difference, d2, the r = qs * h_i cutoff) uses
// round-to-nearest intrinsics (no FMA contraction), so with a pair function compiled
// without contraction (nvcc -fmad=false) the results equal the reference's
// reduce<Real> bit for bit.
//
// Requirements: the pair function (BasicPairKernel::fn, or K::pair for other kernel
// types) and the postamble must be callable on the device (extended __host__
// __device__ lambdas: nvcc --extended-lambda; std::array needs
// --expt-relaxed-constexpr). Gather stores only (symmetric stores: InputError).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <functional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "sfcnl/neighbor_store.hpp"
#include "sfcnl/pair_kernel.hpp"
#include "sfcnl_cu.h"

namespace sfcnl {
namespace gpu {
namespace dev {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double rnd(double a) { return rint(a); }
__device__ __forceinline__ float rnd(float a) { return rintf(a); }

// detail::min_image (reduce.hpp:23-27)
template <class Real>
__device__ __forceinline__ Real min_image(Real d, Real len) {
    if (len > Real(0)) d = sub(d, mul(len, rnd(div(d, len))));
    return d;
}

// reduce_op (pair_kernel.hpp:46-49)
template <class Real>
__device__ __forceinline__ Real reduce_op(int r, Real acc, Real v) {
    return r == 0 ? add(acc, v) : (r == 1 ? (acc < v ? acc : v) : (acc > v ? acc : v));
}

template <class K, class = void>
struct HasFn : std::false_type {};
template <class K>
struct HasFn<K, std::void_t<decltype(&K::fn)>> : std::true_type {};

// decode errors: the lowest super-cluster's wins (parallel_for in order,
// reduce.hpp:217-220); messages as decode_entry_indices / decode_into
enum { kMsgMaskSlice = 1, kMsgTruncMask = 2, kMsgTruncNib = 3, kMsgTrailing = 4, kMsgRawLen = 5 };
struct Err {
    unsigned long long key;  // (sc << 8) | message
    unsigned long long offset;
};
__device__ __forceinline__ void raise(Err* e, uint64_t sc, int msg, uint64_t off) {
    const unsigned long long k = ((unsigned long long)sc << 8) | unsigned(msg);
    if (k < atomicMin(&e->key, k)) e->offset = off;
}

template <class Real, class K, std::size_t NIn, std::size_t NOut>
__global__ void __launch_bounds__(64) k_user_pass(const sfcnl_cu_device_view v, const K kernel,
                                                  const std::array<const double*, NIn> in,
                                                  const std::array<int, NOut> red, const std::array<Real, NOut> ident,
                                                  const Real qs, const std::array<Real*, NOut> out,
                                                  uint32_t* __restrict__ cnt, Err* err) {
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    __shared__ unsigned long long s_pos, s_running;
    const uint32_t t = threadIdx.x;
    const uint32_t ci = v.ci, cj = v.cj, icl_per_sc = 64 / ci, mask_bytes = (icl_per_sc + 7) / 8;
    const uint64_t n = v.n, num_icl = (n + ci - 1) / ci;
    const Real len3[3] = {Real(v.box_len[0]), Real(v.box_len[1]), Real(v.box_len[2])};
    for (uint64_t sc = blockIdx.x; sc < v.num_sc; sc += gridDim.x) {
        const uint64_t i = sc * 64 + t;
        const uint32_t b = t / ci;
        const uint64_t gi = sc * icl_per_sc + b;
        const bool active = i < n && gi < num_icl;
        std::array<Real, NOut> vals = ident;
        uint32_t c = 0;
        PairArgs<Real> args;
        std::array<Real, NIn> in_i{};
        Real r = Real(0);
        if (active) {
            args.i = i;
            args.pos_i = {Real(v.x[i]), Real(v.y[i]), Real(v.z[i])};
            args.h_i = Real(v.h[i]);
            for (std::size_t k = 0; k < NIn; ++k) in_i[k] = Real(in[k][i]);
            r = mul(qs, args.h_i);
        }
        const uint32_t count = v.counts[sc];
        const uint64_t begin = v.offsets[sc], end = v.offsets[sc + 1];
        const uint64_t mb = uint64_t(count) * mask_bytes;
        const uint8_t* records = v.blob + begin;
        const uint8_t* data = records + mb;
        const uint64_t size = end - begin - mb;
        bool bad = false;
        if (count) {
            if (begin + mb > end) {
                if (t == 0) raise(err, sc, kMsgMaskSlice, begin);
                bad = true;
            } else if (!v.compress && size != uint64_t(count) * 4) {
                if (t == 0) raise(err, sc, kMsgRawLen, size);
                bad = true;
            }
        }
        if (t == 0) s_pos = 0, s_running = 0;
        for (uint32_t first = 0; !bad && first < count; first += uint32_t(v.w)) {
            const uint32_t len = min(uint32_t(v.w), count - first);
            __syncthreads();  // the previous block is consumed
            if (t == 0) {
                int res = int(len);
                if (v.compress) {
                    uint64_t pos = s_pos, running = s_running;
                    bool half = false;
                    const uint32_t wb = uint32_t(v.w) / 8;
                    if (pos + wb > size) {
                        raise(err, sc, kMsgTruncMask, pos);
                        res = -1;
                    } else {
                        unsigned long long bm = 0;
                        for (uint32_t q = 0; q < wb; ++q) bm |= (unsigned long long)data[pos + q] << (8 * q);
                        pos += wb;
                        const unsigned long long used = len == 64 ? bm : (bm & ((1ull << len) - 1ull));
                        const int set = __popcll(used);
                        uint8_t info[64];
                        auto take = [&](uint8_t& nib) {
                            if (pos >= size) return false;
                            if (half) {
                                half = false;
                                nib = uint8_t(data[pos++] >> 4);
                            } else {
                                half = true;
                                nib = uint8_t(data[pos] & 0x0f);
                            }
                            return true;
                        };
                        for (int s = 0; s < set && res >= 0; ++s)
                            if (!take(info[s])) raise(err, sc, kMsgTruncNib, pos), res = -1;
                        int at = 0;
                        for (uint32_t k = 0; k < len && res >= 0; ++k) {
                            unsigned long long diff = 1;
                            if ((used >> k) & 1ull) {
                                const uint8_t nib = info[at++];
                                if (nib >= 8) {
                                    diff = nib - 6;
                                } else {
                                    diff = 0;
                                    for (int p = 0; p <= nib && res >= 0; ++p) {
                                        uint8_t d = 0;
                                        if (!take(d)) raise(err, sc, kMsgTruncNib, pos), res = -1;
                                        diff = (diff << 4) | d;
                                    }
                                }
                            }
                            running += diff;
                            s_idx[k] = uint32_t(running - 1);
                        }
                        if (half) ++pos;  // align
                        if (res >= 0 && first + len == count && pos != size) raise(err, sc, kMsgTrailing, pos), res = -1;
                    }
                    s_pos = pos, s_running = running;
                } else {
                    for (uint32_t k = 0; k < len; ++k) {
                        const uint8_t* p = data + 4ull * (first + k);
                        s_idx[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
                    }
                }
                for (uint32_t k = 0; k < len; ++k) {
                    unsigned long long m = 0;
                    for (uint32_t q = 0; q < mask_bytes; ++q)
                        m |= (unsigned long long)records[uint64_t(first + k) * mask_bytes + q] << (8 * q);
                    s_msk[k] = m;
                }
                s_len = res;
            }
            __syncthreads();
            const int l = s_len;
            if (l < 0) {
                bad = true;
                break;
            }
            if (!active) continue;
            for (int e = 0; e < l; ++e) {
                if (!((s_msk[e] >> b) & 1ull)) continue;
                const uint64_t jb = uint64_t(s_idx[e]) * cj, je = min(jb + cj, n);
                for (uint64_t j = jb; j < je; ++j) {
                    if (i == j) continue;
                    args.pos_j = {Real(v.x[j]), Real(v.y[j]), Real(v.z[j])};
                    args.dx = {min_image(sub(args.pos_i.x, args.pos_j.x), len3[0]),
                               min_image(sub(args.pos_i.y, args.pos_j.y), len3[1]),
                               min_image(sub(args.pos_i.z, args.pos_j.z), len3[2])};
                    args.d2 = add(add(mul(args.dx.x, args.dx.x), mul(args.dx.y, args.dx.y)), mul(args.dx.z, args.dx.z));
                    args.h_j = Real(v.h[j]);
                    if (args.d2 > mul(r, r)) continue;
                    args.j = j;
                    std::array<Real, NIn> in_j{};
                    for (std::size_t k = 0; k < NIn; ++k) in_j[k] = Real(in[k][j]);
                    std::array<Real, NOut> pv;
                    if constexpr (HasFn<K>::value) pv = kernel.fn(args, in_i, in_j);
                    else pv = kernel.pair(args, in_i, in_j);
                    for (std::size_t o = 0; o < NOut; ++o) vals[o] = reduce_op(red[o], vals[o], pv[o]);
                    ++c;
                }
            }
        }
        __syncthreads();  // thread 0's decode state is reused by the next SC
        if (!active || bad) continue;
        if constexpr (K::has_postamble) {
            if constexpr (HasFn<K>::value) kernel.post(std::size_t(i), vals, c);
            else kernel.postamble(std::size_t(i), vals, c);
        }
        for (std::size_t o = 0; o < NOut; ++o) out[o][i] = vals[o];
        cnt[i] = c;
    }
}

[[noreturn]] inline void throw_decode(unsigned long long key, unsigned long long off) {
    static const char* const msgs[] = {"", "blob slice too short for bitmasks", "truncated bitmask",
                                       "truncated nibble stream", "trailing bytes in index blob",
                                       "raw index blob length mismatch"};
    const unsigned m = unsigned(key & 255u);
    throw DecodeError(m < 6 ? msgs[m] : "decode error", std::size_t(off));
}

inline void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("sfcnl B200 user pass: ") + cudaGetErrorString(e));
}

}  // namespace dev

/// reduce<Real, K> for user kernels: the reference's reduce loop on the device.
template <class Real, class K>
ReduceResult<Real> reduce_user(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store,
                               const K& kernel, const PassConfig& cfg) {
    constexpr std::size_t NIn = K::num_inputs;
    constexpr std::size_t NOut = K::num_outputs;
    static_assert(std::is_same_v<Real, double> || std::is_same_v<Real, float>, "Real must be double or float");
    const std::size_t n = ps.size();
    std::vector<std::string> fields;
    for (std::size_t k = 0; k < NIn; ++k) fields.emplace_back(kernel.inputs[k]);
    std::array<int, NOut> red{};
    std::array<Real, NOut> ident{};
    ReduceResult<Real> res;
    for (std::size_t o = 0; o < NOut; ++o) {
        red[o] = int(kernel.outputs[o].reduction);
        ident[o] = reduction_identity<Real>(kernel.outputs[o].reduction);
        res.names.emplace_back(kernel.outputs[o].name);
        res.outputs.emplace_back(n, ident[o]);
    }
    res.neighbor_count.assign(n, 0);
    if (store.n != n) throw InputError("reduce: store/particle-set size mismatch");
    if (cfg.query_scale > store.build.build_radius_scale)
        throw InputError("reduce: query_scale exceeds the store's build radius scale");
    if (n == 0) return res;
    with_device_pass(ps, box, store, fields, cfg,
                     [&](const sfcnl_cu_device_view& v, const std::vector<const double*>& fp) {
                         cudaStream_t st = static_cast<cudaStream_t>(v.stream);
                         std::array<const double*, NIn> in{};
                         for (std::size_t k = 0; k < NIn; ++k) in[k] = fp[k];
                         void* buf = nullptr;
                         const std::size_t obytes = NOut * n * sizeof(Real), cbytes = n * sizeof(uint32_t);
                         dev::cuda_check(cudaMallocAsync(&buf, obytes + cbytes + sizeof(dev::Err) + 16, st));
                         std::array<Real*, NOut> out{};
                         for (std::size_t o = 0; o < NOut; ++o) out[o] = static_cast<Real*>(buf) + o * n;
                         uint32_t* cnt = reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + obytes);
                         auto* err = reinterpret_cast<dev::Err*>(static_cast<char*>(buf) + ((obytes + cbytes + 15) & ~std::size_t(15)));
                         dev::cuda_check(cudaMemsetAsync(err, 0xff, sizeof(dev::Err), st));
                         int sms = 148;
                         cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
                         const unsigned grid = unsigned(std::min<uint64_t>(v.num_sc, uint64_t(sms) * 16));
                         dev::k_user_pass<Real, K, NIn, NOut><<<grid, 64, 0, st>>>(v, kernel, in, red, ident, Real(cfg.query_scale),
                                                                                  out, cnt, err);
                         dev::cuda_check(cudaGetLastError());
                         dev::Err he{};
                         for (std::size_t o = 0; o < NOut; ++o)
                             dev::cuda_check(cudaMemcpyAsync(res.outputs[o].data(), out[o], n * sizeof(Real),
                                                             cudaMemcpyDeviceToHost, st));
                         dev::cuda_check(cudaMemcpyAsync(res.neighbor_count.data(), cnt, cbytes, cudaMemcpyDeviceToHost, st));
                         dev::cuda_check(cudaMemcpyAsync(&he, err, sizeof(he), cudaMemcpyDeviceToHost, st));
                         dev::cuda_check(cudaFreeAsync(buf, st));
                         dev::cuda_check(cudaStreamSynchronize(st));
                         if (he.key != ~0ull) dev::throw_decode(he.key, he.offset);
                     });
    return res;
}

}  // namespace gpu
}  // namespace sfcnl
