// B200 drop-in: list build (reference: proj/include/sfcnl/neighbor_build.hpp).
#pragma once

#include "sfcnl/neighbor_store.hpp"
#include "sfcnl/octree.hpp"

namespace sfcnl {

/// GPU: traversal, masks and nibble encode; the result is byte-identical to the
/// reference store. `threads` is accepted for API compatibility and ignored.
NeighborStore build_neighbor_store(const ParticleSet& ps, const SimulationBox& box, const Octree& tree,
                                   const BuildParams& bp, int threads = 1);

}  // namespace sfcnl
