// B200 drop-in: thread-count helper (reference: proj/include/sfcnl/parallel.hpp). The
// reference's parallel_for/parallel_ordered are replaced by CUDA grids; only the
// `threads` argument convention survives (accepted, ignored by the GPU path).
#pragma once

#include <thread>

namespace sfcnl {

inline int resolve_threads(int threads) {
    if (threads > 0) return threads;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? int(hw) : 1;
}

}  // namespace sfcnl
