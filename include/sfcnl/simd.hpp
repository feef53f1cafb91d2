// B200 drop-in: ISA selection (reference: proj/include/sfcnl/simd.hpp). Kept for API
// compatibility of PassConfig; the pass always runs on the GPU.
#pragma once

#include <cstdint>

#include "sfcnl/core.hpp"

namespace sfcnl {

enum class Isa : std::uint8_t { automatic, scalar, avx2 };

bool cpu_supports_avx2();
bool compiled_with_avx2();
Isa resolve_isa(Isa requested);
const char* isa_name(Isa isa);

}  // namespace sfcnl
