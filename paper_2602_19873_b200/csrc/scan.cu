// Device exclusive scan (three-phase: tile sums -> scan of tile sums -> apply).
// Used for octree level compaction (u32) and the store offsets (u32 sizes ->
// u64 offsets, neighbor_store.hpp:48). out has n + 1 entries; out[n] = total.
#include "scan.hpp"

namespace sfcnl_cu {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class In, class Out>
__global__ void k_tile_sums(const In* __restrict__ in, uint64_t n, Out* __restrict__ sums) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    Out s = 0;
    for (int k = threadIdx.x; k < kScanTile; k += kScanThreads) {
        const uint64_t i = base + k;
        if (i < n) s += Out(in[i]);
    }
    s = warp_sum(s);
    __shared__ Out ws[kScanThreads / 32];
    if (lane_id() == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        Out t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

// Single block: exclusive scan of the tile sums in place (any length).
template <class Out>
__global__ void k_scan_sums(Out* sums, uint64_t m, Out* total) {
    __shared__ Out ws[33];
    Out carry = 0;
    for (uint64_t base = 0; base < m; base += 1024) {
        const uint64_t i = base + threadIdx.x;
        const Out v = i < m ? sums[i] : Out(0);
        const Out inc = warp_incl_scan(v);
        if (lane_id() == 31) ws[threadIdx.x >> 5] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            Out s = ws[threadIdx.x];
            s = warp_incl_scan(s);
            ws[threadIdx.x] = s;
        }
        __syncthreads();
        const Out excl = carry + (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : Out(0)) + inc - v;
        if (i < m) sums[i] = excl;
        const Out chunk = ws[31];
        __syncthreads();
        carry += chunk;
    }
    if (threadIdx.x == 0) *total = carry;
}

template <class In, class Out>
__global__ void k_apply(const In* __restrict__ in, uint64_t n, const Out* __restrict__ sums,
                        Out* __restrict__ out) {
    __shared__ Out ws[33];
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanItems;
    Out v[kScanItems];
    Out t = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        v[k] = i < n ? Out(in[i]) : Out(0);
        t += v[k];
    }
    const Out inc = warp_incl_scan(t);
    if (lane_id() == 31) ws[threadIdx.x >> 5] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        Out s = threadIdx.x < kScanThreads / 32 ? ws[threadIdx.x] : Out(0);
        s = warp_incl_scan(s);
        ws[threadIdx.x] = s;
    }
    __syncthreads();
    Out run = sums[blockIdx.x] + (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : Out(0)) + inc - t;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
}

template <class In, class Out>
int scan_impl(sfcnl_cu_ctx* c, const In* in, Out* out, uint64_t n) {
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    SFCNL_CUDA_TRY(c->scan_tmp.reserve((tiles + 1) * sizeof(Out)));
    Out* sums = c->scan_tmp.as<Out>();
    if (n == 0) {
        SFCNL_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(Out), c->stream));
        return 0;
    }
    launch(c, k_tile_sums<In, Out>, dim3(unsigned(tiles)), dim3(kScanThreads), 0, in, n, sums);
    launch(c, k_scan_sums<Out>, dim3(1), dim3(1024), 0, sums, tiles, out + n);
    launch(c, k_apply<In, Out>, dim3(unsigned(tiles)), dim3(kScanThreads), 0, in, n,
           (const Out*)sums, out);
    SFCNL_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace

int excl_scan(sfcnl_cu_ctx* c, const uint32_t* in, uint32_t* out, uint64_t n) {
    return scan_impl<uint32_t, uint32_t>(c, in, out, n);
}
int excl_scan(sfcnl_cu_ctx* c, const uint32_t* in, uint64_t* out, uint64_t n) {
    return scan_impl<uint32_t, uint64_t>(c, in, out, n);
}

}  // namespace sfcnl_cu
