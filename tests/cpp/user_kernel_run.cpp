// Runs the user pair kernels of user_kernels.hpp through reduce<Real> on a set of
// stores and writes every output and neighbour count to argv[1] (raw little-endian:
// per case, per Real, per kernel: outputs then counts). Compiled twice from this one
// file: against the unmodified reference (g++, -Dsfcnl=sfcnl_ref, oracle/_ref) to
// produce tests/golden/user_kernels.bin, and against the B200 drop-in (nvcc) where
// the same calls run the generic device pass (include/sfcnl/gpu_pair_kernel.cuh).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sfcnl/generators.hpp"
#include "sfcnl/hilbert.hpp"
#include "sfcnl/neighbor_build.hpp"
#include "sfcnl/octree.hpp"
#include "sfcnl/reduce.hpp"
#include "user_kernels.hpp"

using namespace sfcnl;

template <class Real, class K>
static void run(FILE* f, const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store, const K& k,
                double qs) {
    PassConfig cfg;
    cfg.query_scale = qs;
    const ReduceResult<Real> r = reduce<Real>(ps, box, store, k, cfg);
    for (const auto& o : r.outputs) std::fwrite(o.data(), sizeof(Real), o.size(), f);
    std::fwrite(r.neighbor_count.data(), 4, r.neighbor_count.size(), f);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 2;
    struct Case {
        int gen;  // 0 uniform, 1 evrard
        std::size_t n;
        double target;
        ClusterParams cp;
        bool compress;
        double scale, qs;
    };
    const Case cases[] = {
        {0, 20000, 80.0, ClusterParams(8, 8, 32), true, 1.0, 1.0},
        {0, 20011, 80.0, ClusterParams(8, 4, 64), true, 1.1, 0.95},
        {1, 12000, 80.0, ClusterParams(8, 8, 32), true, 1.0, 1.0},
        {0, 3001, 40.0, ClusterParams(1, 1, 32), true, 1.0, 1.0},
        {0, 9000, 60.0, ClusterParams(8, 8, 32), false, 1.0, 1.0},
    };
    for (const Case& c : cases) {
        SimulationBox box;
        ParticleSet ps;
        if (c.gen == 0) {
            UniformSpec s;
            s.n = c.n;
            s.density = double(c.n);
            s.target_neighbors = c.target;
            ps = make_uniform(s, box);
        } else {
            EvrardSpec s;
            s.n = c.n;
            s.target_neighbors = c.target;
            ps = make_evrard(s, box);
        }
        const SfcOrder order = sort_by_sfc(ps, box);
        const ParticleSet sorted = apply_sfc_order(ps, order);
        const Octree tree = build_octree(order);
        const NeighborStore store =
            build_neighbor_store(sorted, box, tree, BuildParams(c.cp, ListMode::gather, c.compress, c.scale));
        run<double>(f, sorted, box, store, uk_weighted<double>(), c.qs);
        run<double>(f, sorted, box, store, uk_minmax<double>(), c.qs);
        run<double>(f, sorted, box, store, uk_post<double>(), c.qs);
        run<float>(f, sorted, box, store, uk_weighted<float>(), c.qs);
        run<float>(f, sorted, box, store, uk_minmax<float>(), c.qs);
        run<float>(f, sorted, box, store, uk_post<float>(), c.qs);
    }
    std::fclose(f);
    std::printf("user kernels ok\n");
    return 0;
}
