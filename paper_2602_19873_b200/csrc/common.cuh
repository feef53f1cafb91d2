// Shared device helpers for the sm_100a kernels of the compressed clustered
// neighbor list (build + neighborhood pass).
//
// Exactness contract: the reference is compiled with -ffp-contract=off
// (proj/src/CMakeLists.txt:14), so every fp64 expression that feeds a parity
// decision (SFC grid coordinates, AABB gaps, pair distances, the fp64 pass) is
// written with explicit round-to-nearest intrinsics (__dadd_rn/__dmul_rn/...),
// which nvcc never contracts into FMA. Everything else is free to use FMA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sfcnl_cu.h"

namespace sfcnl_cu {

constexpr int kSC = 64;  // super-cluster size (cluster.hpp:9)

struct Box {
    double lo[3], hi[3], len[3];
    int per[3];
};

// Octree node, byte-compatible with sfcnl::OctreeNode (octree.hpp:11-21).
struct Node {
    uint64_t key_first, key_last;
    uint32_t pbegin, pend;
    int32_t first_child;
    uint8_t depth;
    uint8_t pad[3];
};
static_assert(sizeof(Node) == 32, "Node must stay 32 bytes");

// Axis-aligned box + max radius of a cluster or node; lo/hi follow core.hpp:88-113.
struct Geo {
    double lo[3];
    double hi[3];
    double maxh;
    double pad;
};
static_assert(sizeof(Geo) == 64, "Geo must stay 64 bytes");

// ---------------------------------------------------------------- exact fp64
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// std::min / std::max: first argument wins ties (matters only for signed zeros).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// One axis of periodic_delta (core.hpp:77-85): d -= L * rint(d / L).
// |d| < L/2 (strictly, with margin) gives rint(d/L) == 0 and d - L*0 == d exactly,
// so the division is skipped there; otherwise the reference chain is evaluated.
static __device__ __noinline__ double min_image_wrap(double d, double L) { return dsub(d, dmul(L, rint(ddiv(d, L)))); }
// OL: the rare wrap (and its long division) out of line -- smaller hot kernels (the list
// build: 63.6 -> 59.8 ms at C2); the LJ pass's rare-slot path keeps it inline (faster there)
template <bool OL = true>
__device__ __forceinline__ double min_image_exact(double d, double L, int per) {
    if (!per) return d;
    if (fabs(d) < 0.4999 * L) return d;
    if (OL) return min_image_wrap(d, L);
    return dsub(d, dmul(L, rint(ddiv(d, L))));
}

// Squared minimum-image distance exactly as periodic_delta + Vec3::norm2.
template <bool OL = true>
__device__ __forceinline__ double pair_d2_exact(double xi, double yi, double zi, double xj,
                                                double yj, double zj, const Box& b, double* dx,
                                                double* dy, double* dz) {
    const double ax = min_image_exact<OL>(dsub(xi, xj), b.len[0], b.per[0]);
    const double ay = min_image_exact<OL>(dsub(yi, yj), b.len[1], b.per[1]);
    const double az = min_image_exact<OL>(dsub(zi, zj), b.len[2], b.per[2]);
    if (dx) *dx = ax, *dy = ay, *dz = az;
    return dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az));
}

// interval_interval_gap (core.hpp:132-135)
__device__ __forceinline__ double ii_gap(double alo, double ahi, double blo, double bhi) {
    const double g = dsub(smax(alo, blo), smin(ahi, bhi));
    return g > 0 ? g : 0.0;
}

__device__ __forceinline__ bool geo_empty(const Geo& a) { return a.lo[0] > a.hi[0]; }

// aabb_dist_sq (core.hpp:152-165), bit-exact.
__device__ __forceinline__ double aabb_dist_sq(const Geo& a, const Geo& b, const Box& bx) {
    if (geo_empty(a) || geo_empty(b)) return __longlong_as_double(0x7ff0000000000000LL);
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double g = ii_gap(a.lo[d], a.hi[d], b.lo[d], b.hi[d]);
        if (bx.per[d]) {
            const double L = bx.len[d];
            g = smin(g, ii_gap(a.lo[d], a.hi[d], dsub(b.lo[d], L), dsub(b.hi[d], L)));
            g = smin(g, ii_gap(a.lo[d], a.hi[d], dadd(b.lo[d], L), dadd(b.hi[d], L)));
        }
        s = dadd(s, dmul(g, g));
    }
    return s;
}

__device__ __forceinline__ void geo_init(Geo& a) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    a.lo[0] = a.lo[1] = a.lo[2] = inf;
    a.hi[0] = a.hi[1] = a.hi[2] = -inf;
    a.maxh = 0.0;
    a.pad = 0.0;
}

// Aabb::extend(Vec3) (core.hpp:96-101)
__device__ __forceinline__ void geo_extend_pt(Geo& a, double x, double y, double z) {
    a.lo[0] = smin(a.lo[0], x), a.hi[0] = smax(a.hi[0], x);
    a.lo[1] = smin(a.lo[1], y), a.hi[1] = smax(a.hi[1], y);
    a.lo[2] = smin(a.lo[2], z), a.hi[2] = smax(a.hi[2], z);
}

// Aabb::extend(Aabb) (core.hpp:103-107): skip empty, extend(lo), extend(hi).
__device__ __forceinline__ void geo_extend(Geo& a, const Geo& o) {
    if (geo_empty(o)) return;
    geo_extend_pt(a, o.lo[0], o.lo[1], o.lo[2]);
    geo_extend_pt(a, o.hi[0], o.hi[1], o.hi[2]);
}

// compile-time bool tag for generic lambdas (template specialisation of a loop body)
template <bool B>
struct BoolC {
    static constexpr bool value = B;
};

template <class T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return b < a ? b : a; }

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, v, o);
        if ((int)lane_id() >= o) v += t;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_fmax(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float warp_fmin(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024).
// `scratch` must hold 33 uint32. Returns the exclusive prefix; *total = block sum.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch,
                                                    uint32_t* total) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned nwarps = (blockDim.x + 31) >> 5;
    const uint32_t inc = warp_incl_scan(v);
    if (lane == 31) scratch[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < nwarps ? scratch[lane] : 0u;
        s = warp_incl_scan(s);
        if (lane < nwarps) scratch[lane] = s;
        if (lane == nwarps - 1) scratch[32] = s;
    }
    __syncthreads();
    const uint32_t excl = (warp ? scratch[warp - 1] : 0u) + inc - v;
    *total = scratch[32];
    __syncthreads();
    return excl;
}

// ---------------------------------------------------------------- errors
// Device-side error record; the first (lowest-rank) error wins.
// code = (status << 4) | message index; the driver maps it to SFCNL_* + text.
struct DevError {
    unsigned long long key;  // (rank << 8) | code, atomicMin
    unsigned long long offset;
};

__device__ __forceinline__ void raise_error(DevError* e, uint64_t rank, int status, int msg,
                                            uint64_t offset) {
    const unsigned long long k =
        ((unsigned long long)rank << 8) | (unsigned)((status << 4) | (msg & 15));
    const unsigned long long old = atomicMin(&e->key, k);
    if (k < old) e->offset = offset;  // benign race: offset of some minimal-rank error
}

}  // namespace sfcnl_cu

#define SFCNL_CUDA_TRY(expr)                                                  \
    do {                                                                      \
        cudaError_t _e = (expr);                                              \
        if (_e != cudaSuccess) return ::sfcnl_cu::cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)
