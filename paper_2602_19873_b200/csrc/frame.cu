// Cluster-frame copy of the sorted positions: the fp32 staging format shared by the
// list build and the SPH-density / count pass.
//
// For j-cluster J (cj consecutive sorted particles) with origin c_J = its first
// particle, every particle p of J stores off_p = fl32(minimage(x_p - c_J)) per axis
// plus an optional fp32 payload (the mass), as one float4. A kernel that works in the
// frame of a super-cluster with origin o stages particle p as
//     s_p = fl32( fl32(minimage(c_J - o)) + off_p ),
// one fp64 difference per j-cluster and one fp32 add per coordinate instead of an fp64
// load + difference + minimum image per coordinate. |s_p - (x_p - o)| <=
// 2^-24 (|shift| + |off_p| + |s_p|) <= 2^-23 (|s_p| + |off_p|) (+ fp64 rounding far
// below the guard margins), which the callers' guard bands account for. The global
// maximum |off| per axis (X) bounds the image ambiguity of the per-cluster shift:
// callers treat a super-cluster as unsafe when max|rel_i| + r_max + X >= 0.49 L. The
// per-cluster maximum |off| (xcl) bounds the staging error of a given cluster.
#include "ctx.hpp"

namespace sfcnl_cu {
namespace {

// Clusters [c_lo, c_hi) plus those flagged in jflags (domain decomposition: the
// rank's own range and its halo; other slots of the global-index arrays are stale).
__global__ void k_frame(uint64_t n, uint32_t cj, const double* __restrict__ x, const double* __restrict__ y,
                        const double* __restrict__ z, const double* __restrict__ m, Box box, uint64_t c_lo,
                        uint64_t c_hi, const uint8_t* __restrict__ jflags, float4* __restrict__ frame,
                        unsigned* __restrict__ xmax, unsigned* __restrict__ xcl) {
    float ax = 0.f, ay = 0.f, az = 0.f;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t cl = p / cj;
        if ((cl < c_lo || cl >= c_hi) && !(jflags && jflags[cl])) continue;
        const uint64_t c0 = cl * cj;
        const double v[3] = {x[p], y[p], z[p]}, o[3] = {x[c0], y[c0], z[c0]};
        float f[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double r = dsub(v[d], o[d]);
            if (box.per[d]) {
                const double L = box.len[d];
                if (r > 0.5 * L) r = dsub(r, L);
                else if (r < -0.5 * L) r = dadd(r, L);
            }
            f[d] = float(r);
        }
        ax = fmaxf(ax, fabsf(f[0])), ay = fmaxf(ay, fabsf(f[1])), az = fmaxf(az, fabsf(f[2]));
        frame[p] = make_float4(f[0], f[1], f[2], m ? float(m[p]) : 0.f);
        // per-cluster max |offset| (non-negative floats order like their bits)
        atomicMax(xcl + cl, __float_as_uint(fmaxf(fabsf(f[0]), fmaxf(fabsf(f[1]), fabsf(f[2])))));
    }
    ax = warp_fmax(ax), ay = warp_fmax(ay), az = warp_fmax(az);
    if (lane_id() == 0) {  // non-negative floats order like their bit patterns
        atomicMax(xmax + 0, __float_as_uint(ax));
        atomicMax(xmax + 1, __float_as_uint(ay));
        atomicMax(xmax + 2, __float_as_uint(az));
    }
}

}  // namespace

int run_frame(sfcnl_cu_ctx* c, uint32_t cj, const double* m, uint64_t p_lo, uint64_t p_hi, const uint8_t* jflags) {
    const uint64_t n = c->sorted.n;
    if (p_hi > n) p_hi = n;
    const uint64_t c_lo = p_lo / cj, c_hi = (p_hi + cj - 1) / cj;
    SFCNL_CUDA_TRY(c->frame.reserve(std::max<uint64_t>(n, 1) * sizeof(float4)));
    SFCNL_CUDA_TRY(c->frame_x.reserve(4 * sizeof(unsigned)));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->frame_x.p, 0, 4 * sizeof(unsigned), c->stream));
    const uint64_t ncl = (n + cj - 1) / cj;
    SFCNL_CUDA_TRY(c->frame_xcl.reserve(std::max<uint64_t>(ncl, 1) * sizeof(unsigned)));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->frame_xcl.p, 0, std::max<uint64_t>(ncl, 1) * sizeof(unsigned), c->stream));
    if (n) {
        const int grid = int(std::min<uint64_t>((n + 255) / 256, uint64_t(c->num_sms) * 16));
        launch(c, k_frame, dim3(grid), dim3(256), 0, n, cj, c->sorted.x.as<const double>(), c->sorted.y.as<const double>(),
               c->sorted.z.as<const double>(), m, c->sorted.box, c_lo, c_hi, jflags, c->frame.as<float4>(),
               c->frame_x.as<unsigned>(), c->frame_xcl.as<unsigned>());
    }
    return 0;
}

}  // namespace sfcnl_cu
