// B200 drop-in: the neighborhood pass (reference: proj/include/sfcnl/reduce.hpp).
//
// reduce<Real, K> consults gpu::PassEval<K> (the whole-pass analogue of the
// reference's per-entry simd::EntryEval<K> hook, simd.hpp:50-54). The built-in
// kernels run on the B200: Real = double is the fp64 pass (bit-equal to the
// reference's reduce<double> for gather stores), Real = float is the mixed pass
// (exact neighbour set, values within 1e-5 of fp64). User kernels (make_pair_kernel)
// run as a generic device pass instantiated in the caller's CUDA translation unit
// (gpu_pair_kernel.cuh); in a host-only translation unit they are a compile error:
// there is no CPU fallback on this path.
#pragma once

#include <functional>
#include <string>
#include <type_traits>
#include <vector>

#include "sfcnl/builtin_kernels.hpp"
#include "sfcnl/cluster.hpp"
#include "sfcnl/neighbor_store.hpp"
#include "sfcnl/pair_kernel.hpp"
#include "sfcnl_cu.h"

namespace sfcnl {

namespace gpu {

template <class K>
struct PassEval {
    static constexpr bool available = false;
};
template <class Real>
struct PassEval<CountKernel<Real>> {
    static constexpr bool available = true;
    static constexpr int kind = 0;
};
template <class Real>
struct PassEval<SphDensityKernel<Real>> {
    static constexpr bool available = true;
    static constexpr int kind = 1;
};
template <class Real, bool Coulomb>
struct PassEval<LjKernel<Real, Coulomb>> {
    static constexpr bool available = true;
    static constexpr int kind = Coulomb ? 3 : 2;
};

struct PassRequest {
    int kind = 0;
    int precision = 0;  // 0 fp64, 1 mixed
    double query_scale = 1.0, epsilon = 1.0, sigma = 1.0, coulomb_k = 0.0;
};

/// Runs the pass on the process's default B200 context; outputs are fp64.
void run_pass(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store, const PassRequest& req,
              std::vector<std::vector<double>>& outputs, std::vector<std::uint32_t>& neighbor_count);

/// User pair kernels: uploads the particle set (+ the named input fields) and the store
/// to the default context and calls fn with its device view under the context lock.
void with_device_pass(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store,
                      const std::vector<std::string>& fields, const PassConfig& cfg,
                      const std::function<void(const sfcnl_cu_device_view&, const std::vector<const double*>&)>& fn);

}  // namespace gpu
}  // namespace sfcnl

// user pair kernels (make_pair_kernel / BasicPairKernel): a device pass compiled in the
// caller's CUDA translation unit (gpu_pair_kernel.cuh); host-only callers get a compile error
#ifdef __CUDACC__
#include "sfcnl/gpu_pair_kernel.cuh"
#endif

namespace sfcnl {

template <class K>
struct UserKernelNeedsCuda : std::false_type {};

template <class Real = double, class K>
ReduceResult<Real> reduce(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store,
                          const K& kernel, const PassConfig& cfg = {}) {
    if constexpr (!gpu::PassEval<K>::available) {
#ifdef __CUDACC__
        return gpu::reduce_user<Real>(ps, box, store, kernel, cfg);
#else
        static_assert(UserKernelNeedsCuda<K>::value,
                      "sfcnl B200 drop-in: user pair kernels run as a device pass compiled in a CUDA "
                      "translation unit (nvcc; the pair function must be __device__-callable, e.g. an "
                      "extended __host__ __device__ lambda)");
        return {};
#endif
    } else {
    gpu::PassRequest req;
    req.kind = gpu::PassEval<K>::kind;
    req.precision = std::is_same_v<Real, float> ? 1 : 0;
    req.query_scale = cfg.query_scale;
    if constexpr (gpu::PassEval<K>::kind >= 2) {
        req.epsilon = double(kernel.epsilon);
        req.sigma = double(kernel.sigma);
        req.coulomb_k = double(kernel.coulomb_k);
    }
    std::vector<std::vector<double>> outs;
    ReduceResult<Real> res;
    gpu::run_pass(ps, box, store, req, outs, res.neighbor_count);
    for (std::size_t o = 0; o < K::num_outputs; ++o) {
        res.names.emplace_back(kernel.outputs[o].name);
        res.outputs.emplace_back(outs[o].begin(), outs[o].end());
    }
    return res;
    }
}

}  // namespace sfcnl
