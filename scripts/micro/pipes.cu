// Micro-benchmark: per-SM throughput of FFMA, FFMA2, DFMA, DADD, MUFU.SQRT, FMNMX (ops/clk/SM).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 f2fma(f2 a, f2 b, f2 c) { f2 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int OP>
__global__ void k(float* out, int iters, float s) {
    float a[8]; double d[8]; f2 p[8];
    for (int u = 0; u < 8; ++u) { a[u] = threadIdx.x * 1e-3f + u; d[u] = a[u]; p[u] = (f2)__float_as_uint(a[u]) | ((f2)__float_as_uint(a[u]+1) << 32); }
    const f2 ps = (f2)__float_as_uint(s) | ((f2)__float_as_uint(s) << 32);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) a[u] = fmaf(a[u], s, 0.5f);
            if (OP == 1) p[u] = f2fma(p[u], ps, ps);
            if (OP == 2) d[u] = fma(d[u], (double)s, 0.5);
            if (OP == 3) d[u] = d[u] + (double)s;
            if (OP == 4) { float r; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[u])); a[u] = r; }
            if (OP == 5) a[u] = fmaxf(a[u], s);
            if (OP == 6) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[u])); a[u] = r; }
        }
    }
    long long t1 = clock64();
    float acc = 0; for (int u = 0; u < 8; ++u) acc += a[u] + (float)d[u] + __uint_as_float((unsigned)p[u]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = float(t1 - t0);
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    const char* names[] = {"FFMA", "FFMA2(pairs)", "DFMA", "DADD", "MUFU.SQRT", "FMNMX", "MUFU.RCP"};
    int iters = 4096;
    for (int op = 0; op < 7; ++op) {
        void (*f)(float*, int, float) = op==0?k<0>:op==1?k<1>:op==2?k<2>:op==3?k<3>:op==4?k<4>:op==5?k<5>:k<6>;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            f<<<148 * 4, 512>>>(out, iters, 1.0001f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            float cyc; cudaMemcpy(&cyc, out, 4, cudaMemcpyDeviceToHost);
            double ops = 148.0 * 4 * 512 * iters * 8;  // thread-ops (FFMA2: instructions)
            if (rep) printf("%-14s %.3f ms  %.1f G thread-instr/s  per SM per clk @1.965GHz: %.1f\n", names[op], ms, ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
