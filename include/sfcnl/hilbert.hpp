// B200 drop-in: SFC keys and ordering (reference: proj/include/sfcnl/hilbert.hpp).
// sort_by_sfc / apply_sfc_order run on the GPU (K1 keygen + K2 onesweep radix sort,
// K3 gather); the single-key helpers are host functions producing the same keys
// (48-state refactoring of the reference's Skilling transpose, see csrc/sfc_sort.cu).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "sfcnl/core.hpp"

namespace sfcnl {

inline constexpr int kDefaultSfcBits = 21;
inline constexpr int kMaxSfcBits = 21;

using HilbertKey = std::uint64_t;

inline void check_sfc_bits(int bits) {
    if (bits < 1 || bits > kMaxSfcBits) throw InputError("bits per dimension must be in [1, 21]");
}

HilbertKey hilbert_encode(std::uint32_t ix, std::uint32_t iy, std::uint32_t iz, int bits);
std::array<std::uint32_t, 3> hilbert_decode(HilbertKey key, int bits);

inline std::array<std::uint32_t, 3> grid_coords(const Vec3& pos, const SimulationBox& box, int bits) {
    check_sfc_bits(bits);
    const double cells = double(std::uint64_t(1) << bits);
    std::array<std::uint32_t, 3> g{};
    for (int d = 0; d < 3; ++d) {
        if (!std::isfinite(pos[d])) throw InputError("grid_coords: non-finite coordinate");
        double f = (pos[d] - box.lo[d]) / box.length(d) * cells;
        if (f < 0) f = 0;
        double c = std::floor(f);
        if (c > cells - 1) c = cells - 1;
        g[d] = std::uint32_t(c);
    }
    return g;
}

inline HilbertKey sfc_key(const Vec3& pos, const SimulationBox& box, int bits) {
    const auto g = grid_coords(box.wrap(pos), box, bits);
    return hilbert_encode(g[0], g[1], g[2], bits);
}

struct SfcOrder {
    std::vector<HilbertKey> keys;      ///< ascending
    std::vector<std::uint32_t> perm;   ///< sorted slot -> original index
    int bits = kDefaultSfcBits;
    std::size_t size() const { return keys.size(); }
};

/// GPU: keys of every particle + stable ascending order (ties keep original order).
SfcOrder sort_by_sfc(const ParticleSet& ps, const SimulationBox& box, int bits = kDefaultSfcBits);

/// GPU: out[k] = in[order.perm[k]] for x, y, z, h and every field.
ParticleSet apply_sfc_order(const ParticleSet& ps, const SfcOrder& order);

}  // namespace sfcnl
