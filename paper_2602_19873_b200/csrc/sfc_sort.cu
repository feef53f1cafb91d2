// (1) SFC keygen + stable LSD onesweep radix sort + permutation gather.
//
// Replaces sort_by_sfc (hilbert.cpp:8-26) and apply_sfc_order (hilbert.cpp:28-44).
//
// K1 keygen: one thread per particle. Wrap + grid snapping reproduce
//   SimulationBox::wrap (core.hpp:65-73) and grid_coords (hilbert.hpp:94-107) with
//   round-to-nearest fp64 intrinsics (no FMA contraction), then the Hilbert key is
//   produced by a 48-state machine that is an exact refactoring of the reference's
//   Skilling transpose + interleave (hilbert.hpp:20-38, 66-77): per level, the
//   3 input bits index a smem table (state x octant -> 3 key bits, next state).
//   The same pass accumulates the per-pass 8-bit digit histograms of the sort.
//   Bytes/particle: 24 read + 8 key + 4 index written.
// K2 onesweep: 4096-key tiles, warp-level stable ranking with __match_any_sync,
//   decoupled look-back over per-digit tile counts, smem staging so the scatter
//   writes are digit-contiguous. ceil(3*bits/8) passes; passes whose digit is
//   constant are skipped. Stability + identity values => ties keep original order
//   (the std::stable_sort contract, test_hilbert.cpp:133-142).
//   Bytes/particle/pass: 12 read + 12 written.
// K3 gather: out[k] = in[perm[k]] for x,y,z,h and every field, one launch.
#include <algorithm>
#include <vector>

#include "ctx.hpp"

namespace sfcnl_cu {

// ---------------------------------------------------------------- Hilbert table
// State = (axis permutation, flip mask, parity). See hilbert.hpp:20-38: at level q
// the reference reads bit q of each (transformed) axis and then either flips the
// low bits of X[0] or swaps the low bits of X[0] and X[i]; that accumulated map is
// the state. The final Gray-decode + parity pass (hilbert.hpp:32-37) is folded in.
void hilbert_table(uint16_t* table) {
    struct S {
        int perm[3];
        int f;
        int par;
        bool operator==(const S& o) const {
            return perm[0] == o.perm[0] && perm[1] == o.perm[1] && perm[2] == o.perm[2] &&
                   f == o.f && par == o.par;
        }
    };
    std::vector<S> states;
    states.push_back(S{{0, 1, 2}, 0, 0});
    for (size_t s = 0; s < states.size(); ++s) {
        for (int o = 0; o < 8; ++o) {
            const S st = states[s];
            int c[3];
            for (int i = 0; i < 3; ++i) c[i] = ((o >> (2 - st.perm[i])) & 1) ^ ((st.f >> i) & 1);
            const int g0 = c[0], g1 = c[0] ^ c[1], g2 = c[0] ^ c[1] ^ c[2];
            const int out = ((g0 ^ st.par) << 2) | ((g1 ^ st.par) << 1) | (g2 ^ st.par);
            S nx = st;
            nx.par = st.par ^ g2;
            for (int i = 0; i < 3; ++i) {
                if (c[i]) {
                    nx.f ^= 1;
                } else if (i) {
                    std::swap(nx.perm[0], nx.perm[i]);
                    const int b0 = nx.f & 1, bi = (nx.f >> i) & 1;
                    nx.f = (nx.f & ~1 & ~(1 << i)) | bi | (b0 << i);
                }
            }
            size_t k = 0;
            while (k < states.size() && !(states[k] == nx)) ++k;
            if (k == states.size()) states.push_back(nx);
            table[s * 8 + o] = uint16_t(out | (k << 3));
        }
    }
}

namespace {

constexpr int kTableSize = 48 * 8;
constexpr int kBlockKeys = 256;

__device__ __forceinline__ uint64_t hilbert_key(uint32_t gx, uint32_t gy, uint32_t gz, int bits,
                                                const uint16_t* tab) {
    uint32_t st = 0;
    uint64_t key = 0;
    for (int b = bits - 1; b >= 0; --b) {
        const uint32_t o = (((gx >> b) & 1u) << 2) | (((gy >> b) & 1u) << 1) | ((gz >> b) & 1u);
        const uint32_t e = tab[st * 8 + o];
        key = (key << 3) | (e & 7u);
        st = e >> 3;
    }
    return key;
}

// grid_coords(box.wrap(p)) for one axis (core.hpp:65-73, hilbert.hpp:94-107).
// Two exact shortcuts around the fp64 divisions (values unchanged):
//  * wrap: for lo <= p with fl(p - lo) < L, fl(fl(p - lo) / L) < 1 (division is monotone and
//    fl(L / L) = 1), so floor(.) = 0 and p - L * 0 == p: the division is skipped;
//  * cell: cells = 2^bits, so fl(q) * cells is exact and the cell is floor(fl(q) * cells)
//    with q = fl(p - lo) / len. f' = fl(p - lo) * inv_len * cells (inv_len = fl(1 / len)) is
//    within a few ulps of it (|f' - f| < 2^-48 f <= 2^-27 here), so floor(f') is the cell
//    unless f' lies within 2^-20 of an integer; only then is the exact division evaluated.
__device__ __forceinline__ uint32_t grid_axis(double p, const Box& b, int d, double cells, double inv_len) {
    if (b.per[d]) {
        const double L = b.len[d];
        const double r = dsub(p, b.lo[d]);
        if (!(r >= 0.0 && r < L)) {
            p = dsub(p, dmul(L, floor(ddiv(r, L))));
            if (p >= b.hi[d]) p = b.lo[d];
        }
    }
    const double r = dsub(p, b.lo[d]);
    const double fa = dmul(dmul(r, inv_len), cells);
    const double fl_ = floor(fa);
    double c;
    if (fa - fl_ > 9.5367431640625e-07 && fa - fl_ < 1.0 - 9.5367431640625e-07 && fa < cells - 1.0) {
        c = fl_;
    } else {
        double f = dmul(ddiv(r, b.len[d]), cells);
        if (f < 0) f = 0;
        c = floor(f);
        if (c > cells - 1) c = cells - 1;
    }
    if (c < 0) c = 0;
    return uint32_t(c);
}

__global__ void __launch_bounds__(kBlockKeys) k_keygen(uint64_t n, const double* __restrict__ x,
                                                       const double* __restrict__ y,
                                                       const double* __restrict__ z, Box box,
                                                       int bits, int npass,
                                                       const uint16_t* __restrict__ table,
                                                       uint64_t* __restrict__ keys,
                                                       uint32_t* __restrict__ vals,
                                                       uint32_t* __restrict__ hist, DevError* err) {
    __shared__ uint16_t tab[kTableSize];
    __shared__ uint32_t sh[8][256];
    for (int k = threadIdx.x; k < kTableSize; k += blockDim.x) tab[k] = table[k];
    for (int k = threadIdx.x; k < 8 * 256; k += blockDim.x) (&sh[0][0])[k] = 0;
    __syncthreads();
    const double cells = double(uint64_t(1) << bits);
    const double inv_len[3] = {1.0 / box.len[0], 1.0 / box.len[1], 1.0 / box.len[2]};
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double px = x[i], py = y[i], pz = z[i];
        uint64_t key = 0;
        if (!isfinite(px) || !isfinite(py) || !isfinite(pz)) {
            raise_error(err, i, SFCNL_INPUT_ERROR, 1, 0);
        } else {
            key = hilbert_key(grid_axis(px, box, 0, cells, inv_len[0]), grid_axis(py, box, 1, cells, inv_len[1]),
                              grid_axis(pz, box, 2, cells, inv_len[2]), bits, tab);
        }
        keys[i] = key;
        vals[i] = uint32_t(i);
        for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < npass * 256; k += blockDim.x) {
        const uint32_t v = (&sh[0][0])[k];
        if (v) atomicAdd(&hist[k], v);
    }
}

// Exclusive scan of each pass's 256-bin histogram -> global digit bases.
__global__ void k_digit_base(const uint32_t* hist, uint32_t* base, int npass) {
    const int p = blockIdx.x;
    if (p >= npass) return;
    __shared__ uint32_t scratch[33];
    uint32_t total;
    const uint32_t v = hist[p * 256 + threadIdx.x];
    base[p * 256 + threadIdx.x] = block_excl_scan(v, scratch, &total);
}

constexpr int kSortThreads = 256;
#ifndef SFCNL_SORT_ITEMS
#define SFCNL_SORT_ITEMS 12
#endif
constexpr int kSortItems = SFCNL_SORT_ITEMS;  // keys per thread of a 256-thread tile
constexpr int kTile = kSortThreads * kSortItems;
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kSortThreads) k_onesweep(
    const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, const uint32_t* __restrict__ digit_base,
    uint32_t* status, uint32_t* tile_counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* skeys = reinterpret_cast<uint64_t*>(smem_raw);
    uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + kTile);
    __shared__ uint32_t whist[kSortWarps][256];
    __shared__ uint32_t dstart[256];   // tile-local exclusive digit start
    __shared__ uint32_t dglobal[256];  // global destination of the digit's first key in this tile
    __shared__ uint32_t scratch[33];
    __shared__ uint32_t s_tile;

    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int k = threadIdx.x; k < kSortWarps * 256; k += kSortThreads) (&whist[0][0])[k] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = uint64_t(tile) * kTile;

    uint64_t key[kSortItems];
    uint32_t val[kSortItems];
    uint32_t pos[kSortItems];
    const uint64_t wbase = base + uint64_t(warp) * 32 * kSortItems;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint64_t idx = wbase + j * 32 + lane;
        const bool ok = idx < n;
        key[j] = ok ? kin[idx] : ~0ull;
        val[j] = ok ? vin[idx] : 0u;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint64_t idx = wbase + j * 32 + lane;
        const bool ok = idx < n;
        const uint32_t d = ok ? uint32_t((key[j] >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned leader = __ffs(peers) - 1;
        uint32_t prev = 0;
        if (ok && lane == leader) {
            prev = whist[warp][d];
            whist[warp][d] = prev + __popc(peers);
        }
        prev = __shfl_sync(0xffffffffu, prev, leader);
        pos[j] = prev + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // Per digit (thread t): warp-exclusive prefixes and the tile count.
    const uint32_t t = threadIdx.x;
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t c = whist[w][t];
        whist[w][t] = cnt;
        cnt += c;
    }
    volatile uint32_t* st = status;
    st[uint64_t(tile) * 256 + t] = (tile == 0 ? kFlagInc : kFlagAgg) | cnt;
    uint32_t total;
    dstart[t] = block_excl_scan(cnt, scratch, &total);
    // Decoupled look-back for digit t.
    uint32_t excl = 0;
    if (tile > 0) {
        for (int64_t tt = int64_t(tile) - 1; tt >= 0; --tt) {
            uint32_t s;
            do {
                s = st[uint64_t(tt) * 256 + t];
            } while ((s & (kFlagAgg | kFlagInc)) == 0);
            excl += s & kValMask;
            if (s & kFlagInc) break;
        }
        st[uint64_t(tile) * 256 + t] = kFlagInc | (excl + cnt);
    }
    dglobal[t] = digit_base[t] + excl;
    __syncthreads();

#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint64_t idx = wbase + j * 32 + lane;
        if (idx < n) {
            const uint32_t d = uint32_t((key[j] >> shift) & 255u);
            const uint32_t p = dstart[d] + whist[warp][d] + pos[j];
            skeys[p] = key[j];
            svals[p] = val[j];
        }
    }
    __syncthreads();
    const uint32_t valid = uint32_t(tmin<uint64_t>(kTile, n - base));
    for (uint32_t k = threadIdx.x; k < valid; k += kSortThreads) {
        const uint64_t kk = skeys[k];
        const uint32_t d = uint32_t((kk >> shift) & 255u);
        const uint32_t dst = dglobal[d] + (k - dstart[d]);
        kout[dst] = kk;
        vout[dst] = svals[k];
    }
}

// apply_sfc_order (hilbert.cpp:28-44) as two HBM passes: the SoA inputs are packed
// into narr-double records (sequential), then every output particle fetches its
// whole record (one random 8*narr-byte read instead of narr random 8-byte reads).
// Records of narr doubles, packed back to back.
__global__ void k_pack_records(uint64_t n, int narr, int stride, const double* const* __restrict__ src,
                               double* __restrict__ rec) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x)
        for (int a = 0; a < narr; ++a) rec[k * stride + a] = __ldg(src[a] + k);
}

// Records of 4-6 doubles: pack through shared memory so the records leave as contiguous
// 16-byte stores; gather even widths (16-byte aligned records) with 16-byte loads.
#ifndef SFCNL_PERMUTE_V2
#define SFCNL_PERMUTE_V2 1
#endif
template <int NA>
__global__ void __launch_bounds__(256) k_pack_records_v(uint64_t n, const double* const* __restrict__ src,
                                                        double* __restrict__ rec) {
    __shared__ __align__(16) double s[256 * NA];
    for (uint64_t b0 = uint64_t(blockIdx.x) * 256; b0 < n; b0 += uint64_t(gridDim.x) * 256) {
        const uint32_t m = uint32_t(tmin<uint64_t>(256, n - b0));
        if (threadIdx.x < m) {
#pragma unroll
            for (int a = 0; a < NA; ++a) s[threadIdx.x * NA + a] = __ldg(src[a] + b0 + threadIdx.x);
        }
        __syncthreads();
        const ulonglong2* sv = reinterpret_cast<const ulonglong2*>(s);
        ulonglong2* dv = reinterpret_cast<ulonglong2*>(rec + b0 * NA);  // 16-byte aligned: b0 % 256 == 0
        for (uint32_t k = threadIdx.x; k < m * NA / 2; k += 256) dv[k] = sv[k];
        if ((m * NA) & 1u && threadIdx.x == 0) rec[b0 * NA + m * NA - 1] = s[m * NA - 1];  // odd width, odd tail
        __syncthreads();
    }
}

template <int NA>
__global__ void k_gather_records_v(uint64_t n, const uint32_t* __restrict__ perm, const double* __restrict__ rec,
                                   double* const* __restrict__ dst) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const double2* r = reinterpret_cast<const double2*>(rec + uint64_t(perm[k]) * NA);
        double2 v[NA / 2];
#pragma unroll
        for (int a = 0; a < NA / 2; ++a) v[a] = __ldg(r + a);
#pragma unroll
        for (int a = 0; a < NA / 2; ++a) dst[2 * a][k] = v[a].x, dst[2 * a + 1][k] = v[a].y;
    }
}

template <int NA>
__global__ void k_gather_records(uint64_t n, const uint32_t* __restrict__ perm, int narr, int stride,
                                 const double* __restrict__ rec, double* const* __restrict__ dst) {
    const int na = NA > 0 ? NA : narr;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const double* r = rec + uint64_t(perm[k]) * stride;
        if (NA > 0) {
            double v[NA > 0 ? NA : 1];
#pragma unroll
            for (int a = 0; a < NA; ++a) v[a] = __ldg(r + a);
#pragma unroll
            for (int a = 0; a < NA; ++a) dst[a][k] = v[a];
        } else {
            for (int a = 0; a < na; ++a) dst[a][k] = __ldg(r + a);
        }
    }
}

}  // namespace

int run_sort_by_sfc(sfcnl_cu_ctx* c, int bits) {
    if (bits < 1 || bits > 21) return set_error(c, 1, "bits per dimension must be in [1, 21]");
    if (!c->orig.valid) return set_error(c, 1, "sort_by_sfc: no particles set");
    const uint64_t n = c->orig.n;
    if (n >= (1ull << 30)) return set_error(c, 1, "sort_by_sfc: more than 2^30 particles per GPU");
    c->bits = bits;
    c->order_n = n;
    c->has_order = false;
    const int npass = (3 * bits + 7) / 8;
    SFCNL_CUDA_TRY(c->keys.reserve(n * 8));
    SFCNL_CUDA_TRY(c->keys_alt.reserve(n * 8));
    SFCNL_CUDA_TRY(c->perm.reserve(n * 4));
    SFCNL_CUDA_TRY(c->perm_alt.reserve(n * 4));
    SFCNL_CUDA_TRY(c->hist.reserve(8 * 256 * 4));
    SFCNL_CUDA_TRY(c->digit_base.reserve(8 * 256 * 4));
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    SFCNL_CUDA_TRY(c->status.reserve(std::max<uint64_t>(ntiles, 1) * 256 * 4));
    SFCNL_CUDA_TRY(c->tile_counter.reserve(8 * 4));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->hist.p, 0, 8 * 256 * 4, c->stream));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    if (n == 0) {
        c->has_order = true;
        return 0;
    }

    stage_begin(c, kKeygen);
    {
        const int grid = int(std::min<uint64_t>((n + kBlockKeys - 1) / kBlockKeys, uint64_t(c->num_sms) * 8));
        launch(c, k_keygen, dim3(grid), dim3(kBlockKeys), 0, n, c->orig.x.as<const double>(),
               c->orig.y.as<const double>(), c->orig.z.as<const double>(), c->orig.box, bits, npass,
               c->hilbert_table.as<const uint16_t>(), c->keys.as<uint64_t>(), c->perm.as<uint32_t>(),
               c->hist.as<uint32_t>(), c->derr.as<DevError>());
        SFCNL_CUDA_TRY(cudaGetLastError());
    }
    stage_end(c, kKeygen);
    static const char* const kMsgs[] = {"", "grid_coords: non-finite coordinate"};
    {
        const int rc = check_dev_error(c, kMsgs);
        if (rc) return rc;
    }

    stage_begin(c, kSort);
    launch(c, k_digit_base, dim3(npass), dim3(256), 0, (const uint32_t*)c->hist.as<uint32_t>(),
           c->digit_base.as<uint32_t>(), npass);
    std::vector<uint32_t> hist(npass * 256);
    if (int rc_rb = readback(c, hist.data(), c->hist.p, npass * 256 * 4)) return rc_rb;
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const size_t smem = size_t(kTile) * 12;
    SFCNL_CUDA_TRY(cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    for (int p = 0; p < npass; ++p) {
        bool trivial = false;
        for (int d = 0; d < 256; ++d)
            if (hist[p * 256 + d] == n) trivial = true;
        if (trivial) continue;  // every key has the same digit: order unchanged
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->status.p, 0, ntiles * 256 * 4, c->stream));
        SFCNL_CUDA_TRY(cudaMemsetAsync(c->tile_counter.p, 0, 4, c->stream));
        launch(c, k_onesweep, dim3(unsigned(ntiles)), dim3(kSortThreads), smem,
               (const uint64_t*)c->keys.as<uint64_t>(), (const uint32_t*)c->perm.as<uint32_t>(),
               c->keys_alt.as<uint64_t>(), c->perm_alt.as<uint32_t>(), uint32_t(n), 8 * p,
               (const uint32_t*)(c->digit_base.as<uint32_t>() + p * 256), c->status.as<uint32_t>(),
               c->tile_counter.as<uint32_t>());
        SFCNL_CUDA_TRY(cudaGetLastError());
        std::swap(c->keys, c->keys_alt);
        std::swap(c->perm, c->perm_alt);
    }
    stage_end(c, kSort);
    c->has_order = true;
    c->has_tree = false;
    return 0;
}

int run_apply_order(sfcnl_cu_ctx* c, int64_t into) {
    if (!c->has_order || !c->orig.valid || c->order_n != c->orig.n)
        return set_error(c, 1, "apply_sfc_order: permutation size mismatch");
    const uint64_t n = c->orig.n;
    Slot& s = c->sorted;
    std::vector<const double*> src{c->orig.x.as<double>(), c->orig.y.as<double>(),
                                   c->orig.z.as<double>(), c->orig.h.as<double>()};
    std::vector<double*> dst;
    if (into >= 0) {
        // gather into elements [into, into + n) of an allocated (larger) sorted slot
        if (!s.valid || uint64_t(into) + n > s.n)
            return set_error(c, 1, "apply_order_into: sorted slot too small");
        const uint64_t o = uint64_t(into);
        dst = {s.x.as<double>() + o, s.y.as<double>() + o, s.z.as<double>() + o, s.h.as<double>() + o};
        for (auto& f : c->orig.fields) {
            Field* g = s.find(f.name);
            if (!g) return set_error(c, 1, "apply_order_into: sorted slot lacks field " + f.name);
            src.push_back(f.data.as<double>());
            dst.push_back(g->data.as<double>() + o);
        }
    } else {
        s.n = n;
        s.box = c->orig.box;
        SFCNL_CUDA_TRY(s.x.reserve(n * 8));
        SFCNL_CUDA_TRY(s.y.reserve(n * 8));
        SFCNL_CUDA_TRY(s.z.reserve(n * 8));
        SFCNL_CUDA_TRY(s.h.reserve(n * 8));
        dst = {s.x.as<double>(), s.y.as<double>(), s.z.as<double>(), s.h.as<double>()};
        std::vector<Field> newf;
        for (auto& f : c->orig.fields) {
            Field* existing = s.find(f.name);
            Field g;
            g.name = f.name;
            if (existing) g.data = std::move(existing->data);
            SFCNL_CUDA_TRY(g.data.reserve(n * 8));
            src.push_back(f.data.as<double>());
            dst.push_back(g.data.as<double>());
            newf.push_back(std::move(g));
        }
        s.fields = std::move(newf);
        s.valid = true;
        drop_external(c);
    }
    if (n == 0) return 0;
    const int narr = int(src.size());
    SFCNL_CUDA_TRY(c->ptrs.reserve(2 * narr * sizeof(void*)));
    void** tbl = c->ptrs.as<void*>();
    std::vector<void*> host(2 * narr);
    for (int a = 0; a < narr; ++a) host[a] = (void*)src[a], host[narr + a] = dst[a];
    SFCNL_CUDA_TRY(cudaMemcpyAsync(tbl, host.data(), 2 * narr * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    const int stride = narr;  // (64-byte padded records: gather 8.8 instead of 10.8 GB read, but 0.3 ms slower in all)
    SFCNL_CUDA_TRY(c->records.reserve(n * stride * 8));
    stage_begin(c, kPermute);
    const int grid = int(std::min<uint64_t>((n + 255) / 256, uint64_t(c->num_sms) * 16));
    const uint32_t* pm = c->perm.as<uint32_t>();
    const double* rc = c->records.as<double>();
    double* const* dt = (double* const*)(tbl + narr);
    if (SFCNL_PERMUTE_V2 && narr >= 4 && narr <= 6) {
        const int gp = int(std::min<uint64_t>((n + 255) / 256, uint64_t(c->num_sms) * 8));
        const double* const* sp = (const double* const*)tbl;
        if (narr == 4) {
            launch(c, k_pack_records_v<4>, dim3(gp), dim3(256), 0, n, sp, c->records.as<double>());
            launch(c, k_gather_records_v<4>, dim3(grid), dim3(256), 0, n, pm, rc, dt);
        } else if (narr == 5) {  // 40-byte records: 8-byte gather loads
            launch(c, k_pack_records_v<5>, dim3(gp), dim3(256), 0, n, sp, c->records.as<double>());
            launch(c, k_gather_records<5>, dim3(grid), dim3(256), 0, n, pm, narr, stride, rc, dt);
        } else {
            launch(c, k_pack_records_v<6>, dim3(gp), dim3(256), 0, n, sp, c->records.as<double>());
            launch(c, k_gather_records_v<6>, dim3(grid), dim3(256), 0, n, pm, rc, dt);
        }
        SFCNL_CUDA_TRY(cudaGetLastError());
        stage_end(c, kPermute);
        return 0;
    }
    launch(c, k_pack_records, dim3(grid), dim3(256), 0, n, narr, stride, (const double* const*)tbl, c->records.as<double>());
    switch (narr) {
        case 4: launch(c, k_gather_records<4>, dim3(grid), dim3(256), 0, n, pm, narr, stride, rc, dt); break;
        case 5: launch(c, k_gather_records<5>, dim3(grid), dim3(256), 0, n, pm, narr, stride, rc, dt); break;
        case 6: launch(c, k_gather_records<6>, dim3(grid), dim3(256), 0, n, pm, narr, stride, rc, dt); break;
        default: launch(c, k_gather_records<0>, dim3(grid), dim3(256), 0, n, pm, narr, stride, rc, dt); break;
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kPermute);
    return 0;
}

}  // namespace sfcnl_cu
