// B200 drop-in: the neighborhood pass (reference: proj/include/sfcnl/reduce.hpp).
//
// reduce<Real, K> consults gpu::PassEval<K> (the whole-pass analogue of the
// reference's per-entry simd::EntryEval<K> hook, simd.hpp:50-54). The built-in
// kernels run on the B200: Real = double is the fp64 pass (bit-equal to the
// reference's reduce<double> for gather stores), Real = float is the mixed pass
// (exact neighbour set, values within 1e-5 of fp64). Other kernels are rejected at
// compile time: there is no CPU fallback on this path.
#pragma once

#include <type_traits>

#include "sfcnl/builtin_kernels.hpp"
#include "sfcnl/cluster.hpp"
#include "sfcnl/neighbor_store.hpp"
#include "sfcnl/pair_kernel.hpp"

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

}  // namespace gpu

template <class Real = double, class K>
ReduceResult<Real> reduce(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store,
                          const K& kernel, const PassConfig& cfg = {}) {
    static_assert(gpu::PassEval<K>::available,
                  "sfcnl B200 drop-in: only the built-in kernels (count, SPH density, LJ, LJ+Coulomb) run on "
                  "the GPU pass");
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

}  // namespace sfcnl
