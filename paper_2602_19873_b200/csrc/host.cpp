// Host-side (no device work) parts of the C-ABI: the nibble codec used by the
// C++ drop-in's codec:: functions, the Hilbert key helpers and the seeded input
// generators. None of this is on the GPU hot path; it mirrors reference
// interfaces that are pure host utilities.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "sfcnl_cu.h"

namespace sfcnl_cu {
void hilbert_table(uint16_t* table);
}

namespace {

thread_local std::string g_host_err;
thread_local uint64_t g_host_off = 0;

int herr(int code, const std::string& msg, uint64_t off = 0) {
    g_host_err = msg;
    g_host_off = off;
    return code;
}

const uint16_t* table() {
    static uint16_t t[48 * 8];
    static bool init = [] {
        sfcnl_cu::hilbert_table(t);
        return true;
    }();
    (void)init;
    return t;
}

int bit_width(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

}  // namespace

extern "C" {

const char* sfcnl_last_host_error(uint64_t* byte_offset) {
    if (byte_offset) *byte_offset = g_host_off;
    return g_host_err.c_str();
}

// hilbert_encode (hilbert.hpp:66-77) via the 48-state machine equivalent of the
// Skilling transpose (see csrc/sfc_sort.cu).
int sfcnl_hilbert_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint64_t* key) {
    if (bits < 1 || bits > 21) return herr(SFCNL_INPUT_ERROR, "bits per dimension must be in [1, 21]");
    const uint32_t lim = (1u << bits) - 1;
    if (ix > lim || iy > lim || iz > lim) return herr(SFCNL_INPUT_ERROR, "grid coordinate out of range");
    const uint16_t* tab = table();
    uint32_t st = 0;
    uint64_t k = 0;
    for (int b = bits - 1; b >= 0; --b) {
        const uint32_t o = (((ix >> b) & 1u) << 2) | (((iy >> b) & 1u) << 1) | ((iz >> b) & 1u);
        const uint32_t e = tab[st * 8 + o];
        k = (k << 3) | (e & 7u);
        st = e >> 3;
    }
    *key = k;
    return 0;
}

// hilbert_decode (hilbert.hpp:80-90): inverse walk of the same state machine.
int sfcnl_hilbert_decode(uint64_t key, int bits, uint32_t* xyz) {
    if (bits < 1 || bits > 21) return herr(SFCNL_INPUT_ERROR, "bits per dimension must be in [1, 21]");
    if (bits < 21 && key >= (uint64_t(1) << (3 * bits))) return herr(SFCNL_INPUT_ERROR, "Hilbert key out of range");
    static uint16_t inv[48 * 8];  // state x key-octant -> input octant | next << 3
    static bool init = [] {
        const uint16_t* t = table();
        for (int s = 0; s < 48; ++s)
            for (int o = 0; o < 8; ++o) {
                const uint16_t e = t[s * 8 + o];
                inv[s * 8 + (e & 7)] = uint16_t(o | (e & ~7));
            }
        return true;
    }();
    (void)init;
    uint32_t st = 0, x = 0, y = 0, z = 0;
    for (int b = bits - 1; b >= 0; --b) {
        const uint32_t ko = uint32_t(key >> (3 * b)) & 7u;
        const uint32_t e = inv[st * 8 + ko];
        const uint32_t o = e & 7u;
        x |= ((o >> 2) & 1u) << b, y |= ((o >> 1) & 1u) << b, z |= (o & 1u) << b;
        st = e >> 3;
    }
    xyz[0] = x, xyz[1] = y, xyz[2] = z;
    return 0;
}

// codec::encode (nibble_codec.cpp:117-134): per block of w differences, w/8 mask
// bytes then the info nibbles and the MSB-first data nibbles, packed low nibble
// first, byte-padded.
int sfcnl_codec_encode(const uint32_t* idx, uint64_t count, int w, uint8_t* out, uint64_t cap,
                       uint64_t* len) {
    if (w != 32 && w != 64) return herr(SFCNL_INPUT_ERROR, "block width must be 32 or 64");
    std::vector<uint8_t> bytes;
    uint64_t prev = 0;
    for (uint64_t base = 0; base < count; base += uint64_t(w)) {
        const uint64_t n = std::min<uint64_t>(uint64_t(w), count - base);
        uint64_t mask = 0;
        std::vector<uint8_t> info, data;
        for (uint64_t k = 0; k < n; ++k) {
            const uint64_t cur = idx[base + k];
            uint64_t v;
            if (base + k == 0) {
                v = cur + 1;
            } else {
                if (cur <= prev) return herr(SFCNL_INPUT_ERROR, "delta_encode: input not strictly increasing");
                v = cur - prev;
            }
            prev = cur;
            if (v > 0xffffffffull) return herr(SFCNL_INPUT_ERROR, "encode_block: difference exceeds 2^32 - 1");
            if (v == 1) continue;
            mask |= uint64_t(1) << k;
            if (v <= 9) {
                info.push_back(uint8_t(v + 6));
            } else {
                const int nn = (bit_width(v) + 3) / 4;
                info.push_back(uint8_t(nn - 1));
                for (int p = nn - 1; p >= 0; --p) data.push_back(uint8_t((v >> (4 * p)) & 15u));
            }
        }
        for (int b = 0; b < w / 8; ++b) bytes.push_back(uint8_t(mask >> (8 * b)));
        info.insert(info.end(), data.begin(), data.end());
        for (size_t t = 0; t < info.size(); t += 2)
            bytes.push_back(uint8_t((info[t] & 15u) | ((t + 1 < info.size() ? info[t + 1] : 0u) << 4)));
    }
    *len = bytes.size();
    if (bytes.size() <= cap && !bytes.empty()) std::memcpy(out, bytes.data(), bytes.size());
    return 0;
}

// codec::decode_into (nibble_codec.cpp:136-178) with the same DecodeError offsets.
int sfcnl_codec_decode_into(const uint8_t* data, uint64_t size, uint32_t count, int w, uint32_t* out,
                            uint64_t* consumed) {
    if (w != 32 && w != 64) return herr(SFCNL_INPUT_ERROR, "block width must be 32 or 64");
    uint64_t pos = 0, running = 0;
    bool high = false;
    auto take = [&](uint8_t& v) {
        if (pos >= size) return false;
        if (high) {
            v = uint8_t(data[pos++] >> 4);
            high = false;
        } else {
            v = uint8_t(data[pos] & 15u);
            high = true;
        }
        return true;
    };
    for (uint32_t first = 0; first < count;) {
        const uint32_t n = std::min<uint32_t>(uint32_t(w), count - first);
        if (pos + uint64_t(w / 8) > size) return herr(SFCNL_DECODE_ERROR, "truncated bitmask", pos);
        uint64_t bm = 0;
        for (int b = 0; b < w / 8; ++b) bm |= uint64_t(data[pos + b]) << (8 * b);
        pos += uint64_t(w / 8);
        const uint64_t used = n == 64 ? bm : (bm & ((uint64_t(1) << n) - 1));
        uint8_t info[64];
        int ni = 0;
        for (uint32_t k = 0; k < n; ++k)
            if ((used >> k) & 1u)
                if (!take(info[ni++])) return herr(SFCNL_DECODE_ERROR, "truncated nibble stream", pos);
        int at = 0;
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t d = 1;
            if ((used >> k) & 1u) {
                const uint8_t nb = info[at++];
                if (nb >= 8) {
                    d = uint64_t(nb) - 6;
                } else {
                    d = 0;
                    for (int p = 0; p <= nb; ++p) {
                        uint8_t v;
                        if (!take(v)) return herr(SFCNL_DECODE_ERROR, "truncated nibble stream", pos);
                        d = (d << 4) | v;
                    }
                }
            }
            running += d;
            out[first + k] = uint32_t(running - 1);
        }
        first += n;
        if (high) ++pos, high = false;
    }
    *consumed = pos;
    return 0;
}

// make_uniform (generators.cpp:21-45): std::mt19937_64, 53-bit canonical draws.
int sfcnl_make_uniform(uint64_t n, double density, double target, const int32_t* periodic,
                       double h_jitter, uint64_t seed, double* x, double* y, double* z, double* h,
                       double* m, double* q, double* box6) {
    (void)periodic;
    if (n < 1) return herr(SFCNL_INPUT_ERROR, "make_uniform: n must be >= 1");
    if (!(h_jitter >= 0) || h_jitter >= 1) return herr(SFCNL_INPUT_ERROR, "make_uniform: h_jitter must be in [0, 1)");
    if (!(target > 0) || !(density > 0)) return herr(SFCNL_INPUT_ERROR, "uniform_h_for_target: positive inputs required");
    const double pi = 3.141592653589793;
    const double side = std::cbrt(double(n) / density);
    const double h0 = std::cbrt(3.0 * target / (4.0 * pi * density));
    std::mt19937_64 rng(seed);
    auto u = [&] { return double(rng() >> 11) * 0x1.0p-53; };
    for (uint64_t i = 0; i < n; ++i) {
        x[i] = u() * side;
        y[i] = u() * side;
        z[i] = u() * side;
        h[i] = h_jitter > 0 ? h0 * (1.0 + h_jitter * (2.0 * u() - 1.0)) : h0;
    }
    for (uint64_t i = 0; i < n; ++i) {
        if (m) m[i] = 1.0;
        if (q) q[i] = (i % 2 == 0) ? 1.0 : -1.0;
    }
    for (int d = 0; d < 3; ++d) box6[d] = 0.0, box6[3 + d] = side;
    return 0;
}

// make_evrard (generators.cpp:47-82): r = sqrt(u) (1/r density), h from local spacing.
int sfcnl_make_evrard(uint64_t n, double target, int32_t constant_h, const int32_t* periodic,
                      uint64_t seed, double* x, double* y, double* z, double* h, double* m,
                      double* q, double* box6) {
    (void)periodic;
    if (n < 1) return herr(SFCNL_INPUT_ERROR, "make_evrard: n must be >= 1");
    const double pi = 3.141592653589793, R = 1.0, margin = 1.1 * R;
    const double alpha = std::cbrt(3.0 * target / (4.0 * pi));
    const double mean_r = 2.0 / 3.0 * R;
    std::mt19937_64 rng(seed);
    auto u = [&] { return double(rng() >> 11) * 0x1.0p-53; };
    for (uint64_t i = 0; i < n; ++i) {
        const double r = R * std::sqrt(u());
        const double ct = 1.0 - 2.0 * u();
        const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
        const double phi = 2.0 * pi * u();
        x[i] = r * st * std::cos(phi);
        y[i] = r * st * std::sin(phi);
        z[i] = r * ct;
        const double rh = constant_h ? mean_r : r;
        h[i] = alpha * std::cbrt(2.0 * pi * R * R * rh / double(n));
    }
    for (uint64_t i = 0; i < n; ++i) {
        if (m) m[i] = 1.0 / double(n);
        if (q) q[i] = (i % 2 == 0) ? 1.0 : -1.0;
    }
    for (int d = 0; d < 3; ++d) box6[d] = -margin, box6[3 + d] = margin;
    return 0;
}

}  // extern "C"
