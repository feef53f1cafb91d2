// Helpers of the mixed-precision passes (pass_item.cuh, pass_warp.cuh, pass_symf.cuh),
// included by pass.cu inside namespace sfcnl_cu::{anon}: packed f32x2 arithmetic
// (FADD2 / FMUL2 / FFMA2), fp32 predicates as float masks, and the fp64 reference slot
// (rare_slot) that decides guard-band slots. See pass.cu's header for the numerical
// contract.

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
__device__ __forceinline__ float sqrt_ftz(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float fset_lt(float a, float b) {  // 1.0f if a < b else 0.0f
    float r;
    asm("set.lt.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fset_le(float a, float b) {
    float r;
    asm("set.le.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Rare slot: cutoff inside the guard band, or an LJ pair closer than 1.22 sigma
// (force-zero crossing / overflow range): the exact reference predicate and fp64
// kernel value, accumulated into the SC's shared fp64 side sums.
template <int K, bool OL = true>  // OL: min-image wrap out of line (see common.cuh)
__device__ __noinline__ int rare_slot(const PassArgs& A, uint64_t i, uint64_t j, double r2,
                                      double* side) {
    if (i == j) return 0;
    const double xi = A.x[i], yi = A.y[i], zi = A.z[i], hi = A.h[i];
    double dx, dy, dz;
    const double d2 = pair_d2_exact<OL>(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
    if (d2 > r2) return 0;
    double v[4];
    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) return -1;
    constexpr int NO = nout<K>();
#pragma unroll
    for (int o = 0; o < NO; ++o) atomicAdd(side + o, v[o]);
    return 1;
}
