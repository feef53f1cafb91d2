#pragma once
#include "ctx.hpp"

namespace sfcnl_cu {
// Exclusive scans on the context stream; out must hold n + 1 entries (out[n] = total).
int excl_scan(sfcnl_cu_ctx* c, const uint32_t* in, uint32_t* out, uint64_t n);
int excl_scan(sfcnl_cu_ctx* c, const uint32_t* in, uint64_t* out, uint64_t n);
}  // namespace sfcnl_cu
