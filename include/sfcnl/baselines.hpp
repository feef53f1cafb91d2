// B200 drop-in: the full Verlet list baseline (reference: proj/include/sfcnl/baselines.hpp:25-129).
//
// build_full_list derives the classic per-particle CSR list on the GPU from a
// compressed gather store built at `build_scale` (include/sfcnl_cu.h section (5b));
// the list is identical to the reference's (neighbors ascending, exact fp64
// predicate). Gather mode only: a symmetric full list throws InputError. `method`
// and `cap` are accepted and ignored (the result never depended on them).
// reduce_full runs on the GPU for the built-in kernels: Real = double is bit-equal
// to the reference's reduce_full<double>, Real = float is the warp-per-i pass
// (fp64 values, tree sum). The O(n^2) oracles brute_force_pairs / brute_force_counts /
// reduce_direct are test infrastructure of the reference and are not part of the
// drop-in.
#pragma once

#include <cstdint>
#include <vector>

#include "sfcnl/core.hpp"
#include "sfcnl/neighbor_store.hpp"
#include "sfcnl/pair_kernel.hpp"
#include "sfcnl/reduce.hpp"

namespace sfcnl {

inline constexpr std::size_t kDefaultOracleCap = 50000;

enum class FullListMethod { automatic, brute_force, cell_grid };

/// Classic per-particle Verlet list in CSR form, neighbors ascending.
struct FullVerletList {
    ListMode mode = ListMode::gather;
    double build_scale = 1.0;
    std::vector<std::uint64_t> offsets;  ///< size n + 1
    std::vector<std::uint32_t> neighbors;

    std::uint64_t memory_bytes() const {
        return offsets.size() * sizeof(std::uint64_t) + neighbors.size() * sizeof(std::uint32_t);
    }
};

FullVerletList build_full_list(const ParticleSet& ps, const SimulationBox& box, double build_scale,
                               ListMode mode, FullListMethod method = FullListMethod::automatic,
                               std::size_t cap = kDefaultOracleCap);

namespace gpu {
void run_pass_full(const ParticleSet& ps, const SimulationBox& box, const FullVerletList& list, const PassRequest& req,
                   std::vector<std::vector<double>>& outputs, std::vector<std::uint32_t>& neighbor_count);
}  // namespace gpu

template <class Real = double, class K>
ReduceResult<Real> reduce_full(const ParticleSet& ps, const SimulationBox& box, const FullVerletList& list,
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
    gpu::run_pass_full(ps, box, list, req, outs, res.neighbor_count);
    for (std::size_t o = 0; o < K::num_outputs; ++o) {
        res.names.emplace_back(kernel.outputs[o].name);
        res.outputs.emplace_back(outs[o].begin(), outs[o].end());
    }
    return res;
}

}  // namespace sfcnl
