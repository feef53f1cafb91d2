// Micro-benchmark: issue/pipe throughput of common SASS forms (warp-instr per clk per SM).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
#define F2(op) asm volatile(op : "+l"(p[u]) : "l"(q[u]), "l"(q[(u+1)&7]))
template <int OP>
__global__ void k(float* out, int iters, float s, float s2) {
    float a[8], b[8]; f2 p[8], q[8]; unsigned x[8];
    for (int u = 0; u < 8; ++u) { a[u] = threadIdx.x * 1e-3f + u; b[u] = a[u] * s2; x[u] = threadIdx.x + u;
        p[u] = (f2)__float_as_uint(a[u]) | ((f2)__float_as_uint(b[u]) << 32); q[u] = p[u] ^ 0x1234; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) a[u] = fmaf(a[u], b[u], b[(u + 1) & 7]);           // FFMA 3-reg
            if (OP == 1) a[u] = a[u] + b[u];                                 // FADD
            if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[u]) : "l"(q[u]), "l"(q[(u+1)&7]));
            if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[u]) : "l"(q[u]));
            if (OP == 4) a[u] = fmaxf(a[u], b[u]);                           // FMNMX
            if (OP == 5) x[u] = x[u] + x[(u + 3) & 7] + 7;                   // IADD3
            if (OP == 6) x[u] = (x[u] ^ x[(u + 3) & 7]) & 0x5555;            // LOP3
            if (OP == 7) a[u] = (a[u] < b[u]) ? b[(u+1)&7] : a[u];           // FSETP+FSEL
        }
    }
    float acc = 0; for (int u = 0; u < 8; ++u) acc += a[u] + __uint_as_float((unsigned)p[u]) + (float)x[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    const char* names[] = {"FFMA 3reg", "FADD", "FFMA2", "FADD2", "FMNMX", "IADD3", "LOP3", "FSETP+FSEL"};
    int iters = 4096;
    for (int op = 0; op < 8; ++op) {
        void (*f)(float*, int, float, float) = op==0?k<0>:op==1?k<1>:op==2?k<2>:op==3?k<3>:op==4?k<4>:op==5?k<5>:op==6?k<6>:k<7>;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            f<<<148 * 4, 512>>>(out, iters, 1.0001f, 0.999f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double wi = 148.0 * 4 * 16 * iters * 8;  // warp-level statements
            if (rep) printf("%-12s %.3f ms  warp-statements per SM per clk @1.965GHz: %.2f\n", names[op], ms, wi / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
