// Drop-in C++ API for the full Verlet list baseline and the cluster-overhead metric
// (include/sfcnl/baselines.hpp, include/sfcnl/bench.hpp) on the GPU, checked against
// the compressed path through the same API: reduce_full<double> over the full list is
// bit-equal to reduce<double> over the gather store (same pairs, ascending j), the
// unsorted-input list is the sorted one renumbered, cluster_overhead equals the slot
// count restated on the host from the decoded store (bench.cpp:93-122).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <algorithm>
#include <cmath>

#include "doctest.h"
#include "sfcnl/baselines.hpp"
#include "sfcnl/bench.hpp"
#include "sfcnl/generators.hpp"
#include "sfcnl/hilbert.hpp"
#include "sfcnl/neighbor_build.hpp"
#include "sfcnl/octree.hpp"
#include "sfcnl/reduce.hpp"

using namespace sfcnl;

TEST_CASE("full list and reduce_full match the compressed path") {
    UniformSpec spec;
    spec.n = 20000;
    spec.density = 20000.0;
    spec.target_neighbors = 60.0;
    SimulationBox box;
    const ParticleSet ps = make_uniform(spec, box);
    const SfcOrder order = sort_by_sfc(ps, box);
    const ParticleSet sorted = apply_sfc_order(ps, order);
    const Octree tree = build_octree(order);
    const NeighborStore store =
        build_neighbor_store(sorted, box, tree, BuildParams(ClusterParams(8, 8, 32), ListMode::gather, true, 1.0));

    const FullVerletList fl = build_full_list(sorted, box, 1.0, ListMode::gather);
    REQUIRE(fl.offsets.size() == ps.size() + 1);
    CHECK(fl.memory_bytes() == 8 * (ps.size() + 1) + 4 * fl.neighbors.size());
    for (std::size_t i = 0; i < ps.size(); ++i)
        CHECK(std::is_sorted(fl.neighbors.begin() + fl.offsets[i], fl.neighbors.begin() + fl.offsets[i + 1]));

    const auto a = reduce<double>(sorted, box, store, sph_density_kernel<double>());
    const auto b = reduce_full<double>(sorted, box, fl, sph_density_kernel<double>());
    CHECK(a.neighbor_count == b.neighbor_count);
    CHECK(a.outputs[0] == b.outputs[0]);
    const auto c = reduce_full<float>(sorted, box, fl, sph_density_kernel<float>());
    CHECK(c.neighbor_count == a.neighbor_count);
    double worst = 0;
    for (std::size_t i = 0; i < ps.size(); ++i)
        worst = std::max(worst, std::abs(double(c.outputs[0][i]) - a.outputs[0][i]) / a.outputs[0][i]);
    CHECK(worst <= 1e-6);  // ReduceResult<float> stores float

    // unsorted input: the same pairs in the caller's numbering
    const FullVerletList fu = build_full_list(ps, box, 1.0, ListMode::gather);
    REQUIRE(fu.neighbors.size() == fl.neighbors.size());
    bool same = true;
    for (std::size_t s = 0; s < ps.size() && same; ++s) {
        std::vector<std::uint32_t> row;
        for (std::uint64_t k = fl.offsets[s]; k < fl.offsets[s + 1]; ++k) row.push_back(order.perm[fl.neighbors[k]]);
        std::sort(row.begin(), row.end());
        const std::uint32_t i = order.perm[s];
        same = std::equal(row.begin(), row.end(), fu.neighbors.begin() + fu.offsets[i],
                          fu.neighbors.begin() + fu.offsets[i + 1]);
    }
    CHECK(same);

    CHECK_THROWS_AS(build_full_list(sorted, box, 1.0, ListMode::symmetric), InputError);
    PassConfig big;
    big.query_scale = 1.5;
    CHECK_THROWS_AS(reduce_full<double>(sorted, box, fl, count_kernel<double>(), big), InputError);
}

TEST_CASE("cluster_overhead equals the host slot count") {
    UniformSpec spec;
    spec.n = 10000;
    spec.density = 10000.0;
    spec.target_neighbors = 50.0;
    SimulationBox box;
    const ParticleSet ps = make_uniform(spec, box);
    const SfcOrder order = sort_by_sfc(ps, box);
    const ParticleSet sorted = apply_sfc_order(ps, order);
    const Octree tree = build_octree(order);
    const NeighborStore store =
        build_neighbor_store(sorted, box, tree, BuildParams(ClusterParams(8, 4, 64), ListMode::gather, true, 1.0));
    const auto cnt = reduce<double>(sorted, box, store, count_kernel<double>()).neighbor_count;
    std::uint64_t pairs = 0;
    for (auto v : cnt) pairs += v;
    std::uint64_t slots = 0;
    const std::uint64_t n = ps.size();
    for (std::uint64_t sc = 0; sc < store.counts.size(); ++sc)
        for (const NeighborEntry& e : neighbor_clusters(store, sc)) {
            const std::uint64_t jb = std::uint64_t(e.jcluster) * 4, je = std::min<std::uint64_t>(jb + 4, n);
            for (int b = 0; b < 8; ++b)
                if ((e.mask >> b) & 1) {
                    const std::uint64_t ib = (sc * 8 + b) * 8;
                    if (ib < n) slots += (std::min<std::uint64_t>(ib + 8, n) - ib) * (je - jb);
                }
        }
    CHECK(bench::cluster_overhead(store, pairs) == double(slots) / double(pairs));
    CHECK_THROWS_AS(bench::cluster_overhead(store, 0), InputError);
}
