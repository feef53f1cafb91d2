// B200 drop-in: the list-quality metric of the reference's bench harness
// (proj/include/sfcnl/bench.hpp:51, bench.cpp:93-122). The CSV harness itself
// (BenchConfig, run_bench) is out of scope; bench.py / scripts/c4_sweep.py report
// the same metrics.
#pragma once

#include <cstdint>

#include "sfcnl/neighbor_store.hpp"

namespace sfcnl::bench {

/// Pair slots the pass evaluates (sum over entries and set mask bits of
/// |i-cluster| * |j-cluster|) divided by the true directed in-range pairs. Gather
/// stores only. The slot count is a device pass over the store.
double cluster_overhead(const NeighborStore& store, std::uint64_t true_directed_pairs);

}  // namespace sfcnl::bench
