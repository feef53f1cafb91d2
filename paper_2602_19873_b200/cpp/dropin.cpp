// The reference's C++ API (include/sfcnl/*.hpp) implemented over the B200 C-ABI
// (include/sfcnl_cu.h). Linked as libsfcnl.so, it replaces the reference's
// libsfcnl.a for callers of the build-and-query path: same declarations, same
// results, GPU-resident hot path. Host-only utilities (codec, store I/O,
// generators, single-key helpers) are plain C++ here.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>

#include "sfcnl/baselines.hpp"
#include "sfcnl/bench.hpp"
#include "sfcnl/builtin_kernels.hpp"
#include "sfcnl/generators.hpp"
#include "sfcnl/hilbert.hpp"
#include "sfcnl/neighbor_build.hpp"
#include "sfcnl/nibble_codec.hpp"
#include "sfcnl/octree.hpp"
#include "sfcnl/reduce.hpp"
#include "sfcnl/simd.hpp"
#include "sfcnl_cu.h"

namespace sfcnl {

namespace {

[[noreturn]] void throw_status(int rc, const char* msg, std::uint64_t off) {
    switch (rc) {
        case SFCNL_INPUT_ERROR: throw InputError(msg);
        case SFCNL_BUILD_ERROR: throw BuildError(msg);
        case SFCNL_DECODE_ERROR: throw DecodeError(msg, std::size_t(off));
        default: throw std::runtime_error(std::string("sfcnl B200: ") + msg);
    }
}

void host_check(int rc) {
    if (!rc) return;
    std::uint64_t off = 0;
    const char* m = sfcnl_last_host_error(&off);
    throw_status(rc, m, off);
}

// Process-wide device context (device = $LOCAL_RANK, else 0), one call at a time.
struct Device {
    sfcnl_cu_ctx* ctx = nullptr;
    std::mutex mu;
    Device() {
        const char* lr = std::getenv("LOCAL_RANK");
        const int dev = lr ? std::atoi(lr) : 0;
        const int rc = sfcnl_cu_ctx_create(dev, &ctx);
        if (rc) throw_status(rc, sfcnl_cu_last_error(nullptr, nullptr), 0);
    }
    ~Device() { sfcnl_cu_ctx_destroy(ctx); }
    void check(int rc) {
        if (!rc) return;
        std::uint64_t off = 0;
        const char* m = sfcnl_cu_last_error(ctx, &off);
        // DecodeError's message already carries the offset suffix from the device side
        if (rc == SFCNL_DECODE_ERROR) {
            std::string s(m);
            const auto p = s.find(" (byte offset");
            throw DecodeError(p == std::string::npos ? s : s.substr(0, p), std::size_t(off));
        }
        throw_status(rc, m, off);
    }
};

Device& device() {
    static Device d;
    return d;
}

sfcnl_box to_box(const SimulationBox& b) {
    sfcnl_box r{};
    for (int d = 0; d < 3; ++d) r.lo[d] = b.lo[d], r.hi[d] = b.hi[d], r.periodic[d] = b.periodic[d] ? 1 : 0;
    return r;
}

void check_lengths(const ParticleSet& ps) {
    const std::size_t n = ps.size();
    if (ps.y.size() != n || ps.z.size() != n || ps.h.size() != n) throw InputError("ParticleSet: array length mismatch");
    for (const auto& f : ps.fields)
        if (f.second.size() != n) throw InputError("ParticleSet: field length mismatch: " + f.first);
}

// Uploads ps (original or sorted slot). Positions need not lie inside `box` for the
// calls that do not interpret them against the box.
void upload(Device& D, const ParticleSet& ps, const SimulationBox& box, bool sorted, bool with_fields) {
    check_lengths(ps);
    const sfcnl_box b = to_box(box);
    const std::size_t n = ps.size();
    auto (*setp)(sfcnl_cu_ctx*, uint64_t, const double*, const double*, const double*, const double*,
                 const sfcnl_box*) -> int = sorted ? sfcnl_cu_set_sorted_particles : sfcnl_cu_set_particles;
    D.check(setp(D.ctx, n, ps.x.data(), ps.y.data(), ps.z.data(), ps.h.data(), &b));
    if (!with_fields) return;
    for (const auto& f : ps.fields)
        D.check((sorted ? sfcnl_cu_set_sorted_field : sfcnl_cu_set_field)(D.ctx, f.first.c_str(), f.second.data()));
}

SimulationBox unit_box() { return SimulationBox({0, 0, 0}, {1, 1, 1}); }

sfcnl_build_params to_params(const BuildParams& bp) {
    sfcnl_build_params p{};
    p.ci = bp.params.ci, p.cj = bp.params.cj, p.w = bp.params.w;
    p.mode = bp.mode == ListMode::symmetric ? 1 : 0;
    p.compress = bp.compress ? 1 : 0;
    p.build_radius_scale = bp.build_radius_scale;
    return p;
}

void upload_tree(Device& D, const Octree& tree) {
    static_assert(sizeof(OctreeNode) == sizeof(sfcnl_node), "OctreeNode layout");
    std::vector<sfcnl_node> nodes(tree.nodes.size());
    for (std::size_t k = 0; k < nodes.size(); ++k) {
        const OctreeNode& s = tree.nodes[k];
        nodes[k] = sfcnl_node{s.key_first, s.key_last, s.particle_begin, s.particle_end, s.first_child, s.depth, {0, 0, 0}};
    }
    D.check(sfcnl_cu_set_octree(D.ctx, nodes.size(), nodes.data(), tree.bits, tree.n));
}

}  // namespace

// ------------------------------------------------------------------ hilbert
HilbertKey hilbert_encode(std::uint32_t ix, std::uint32_t iy, std::uint32_t iz, int bits) {
    HilbertKey k = 0;
    host_check(sfcnl_hilbert_encode(ix, iy, iz, bits, &k));
    return k;
}

std::array<std::uint32_t, 3> hilbert_decode(HilbertKey key, int bits) {
    std::array<std::uint32_t, 3> a{};
    host_check(sfcnl_hilbert_decode(key, bits, a.data()));
    return a;
}

SfcOrder sort_by_sfc(const ParticleSet& ps, const SimulationBox& box, int bits) {
    check_sfc_bits(bits);
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    upload(D, ps, box, false, false);
    D.check(sfcnl_cu_sort_by_sfc(D.ctx, bits));
    SfcOrder o;
    o.bits = bits;
    o.keys.resize(ps.size());
    o.perm.resize(ps.size());
    D.check(sfcnl_cu_get_order(D.ctx, o.keys.data(), o.perm.data()));
    return o;
}

ParticleSet apply_sfc_order(const ParticleSet& ps, const SfcOrder& order) {
    const std::size_t n = ps.size();
    if (order.perm.size() != n) throw InputError("apply_sfc_order: permutation size mismatch");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    upload(D, ps, unit_box(), false, true);
    std::vector<std::uint64_t> keys = order.keys;
    keys.resize(n, 0);
    D.check(sfcnl_cu_set_order(D.ctx, n, keys.data(), order.perm.data(), order.bits));
    D.check(sfcnl_cu_apply_order(D.ctx));
    ParticleSet out;
    out.resize(n);
    D.check(sfcnl_cu_get_sorted(D.ctx, "x", out.x.data()));
    D.check(sfcnl_cu_get_sorted(D.ctx, "y", out.y.data()));
    D.check(sfcnl_cu_get_sorted(D.ctx, "z", out.z.data()));
    D.check(sfcnl_cu_get_sorted(D.ctx, "h", out.h.data()));
    for (const auto& f : ps.fields) {
        auto& v = out.add_field(f.first);
        D.check(sfcnl_cu_get_sorted(D.ctx, f.first.c_str(), v.data()));
    }
    return out;
}

// ------------------------------------------------------------------ octree
Octree build_octree(const SfcOrder& order, std::uint32_t bucket_size) {
    if (bucket_size < 1) throw InputError("build_octree: bucket_size must be >= 1");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const std::size_t n = order.keys.size();
    std::vector<std::uint32_t> perm = order.perm;
    perm.resize(n, 0);
    D.check(sfcnl_cu_set_order(D.ctx, n, order.keys.data(), perm.data(), order.bits));
    std::uint64_t nn = 0;
    D.check(sfcnl_cu_build_octree(D.ctx, bucket_size, &nn));
    std::vector<sfcnl_node> nodes(nn);
    D.check(sfcnl_cu_get_octree(D.ctx, nodes.data()));
    Octree t;
    t.bits = order.bits;
    t.n = std::uint32_t(n);
    t.nodes.resize(nn);
    for (std::size_t k = 0; k < nn; ++k) {
        OctreeNode& d = t.nodes[k];
        d.key_first = nodes[k].key_first, d.key_last = nodes[k].key_last;
        d.particle_begin = nodes[k].particle_begin, d.particle_end = nodes[k].particle_end;
        d.first_child = nodes[k].first_child, d.depth = nodes[k].depth;
    }
    return t;
}

Aabb node_aabb(const Octree& tree, std::int32_t node, const ParticleSet& ps) {
    const OctreeNode& nd = tree.nodes.at(std::size_t(node));
    Aabb box;
    for (std::uint32_t i = nd.particle_begin; i < nd.particle_end; ++i) box.extend(ps.pos(i));
    return box;
}

static void node_geometry(const Octree& tree, const ParticleSet& ps, std::vector<Aabb>* boxes,
                          std::vector<double>* radius) {
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const SimulationBox anywhere({-1e308, -1e308, -1e308}, {1e308, 1e308, 1e308});
    upload(D, ps, anywhere, true, false);
    upload_tree(D, tree);
    const std::size_t nn = tree.nodes.size();
    std::vector<double> lo(3 * nn), hi(3 * nn), rad(nn);
    D.check(sfcnl_cu_node_geometry(D.ctx, lo.data(), hi.data(), rad.data()));
    if (boxes) {
        boxes->resize(nn);
        for (std::size_t k = 0; k < nn; ++k)
            for (int d = 0; d < 3; ++d) (*boxes)[k].lo[d] = lo[3 * k + d], (*boxes)[k].hi[d] = hi[3 * k + d];
    }
    if (radius) *radius = std::move(rad);
}

std::vector<Aabb> compute_node_aabbs(const Octree& tree, const ParticleSet& ps) {
    std::vector<Aabb> b;
    node_geometry(tree, ps, &b, nullptr);
    return b;
}

std::vector<double> compute_node_max_radius(const Octree& tree, const ParticleSet& ps) {
    std::vector<double> r;
    node_geometry(tree, ps, nullptr, &r);
    return r;
}

// ------------------------------------------------------------------ build
NeighborStore build_neighbor_store(const ParticleSet& ps, const SimulationBox& box, const Octree& tree,
                                   const BuildParams& bp, int /*threads*/) {
    check_lengths(ps);
    if (tree.nodes.empty()) throw BuildError("build_neighbor_store: octree/particle-set mismatch");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    upload(D, ps, box, true, false);
    upload_tree(D, tree);
    const sfcnl_build_params p = to_params(bp);
    std::uint64_t nsc = 0, nb = 0;
    D.check(sfcnl_cu_build_store(D.ctx, &p, &nsc, &nb));
    NeighborStore s;
    s.build = bp;
    s.n = ps.size();
    s.counts.resize(nsc);
    s.offsets.resize(nsc + 1);
    s.blob.resize(nb);
    D.check(sfcnl_cu_get_store(D.ctx, s.counts.data(), s.offsets.data(), s.blob.data()));
    return s;
}

// ------------------------------------------------------------------ pass
void gpu::run_pass(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store, const PassRequest& req,
                   std::vector<std::vector<double>>& outputs, std::vector<std::uint32_t>& neighbor_count) {
    const std::size_t n = ps.size();
    if (store.n != n) throw InputError("reduce: store/particle-set size mismatch");
    if (req.query_scale > store.build.build_radius_scale)
        throw InputError("reduce: query_scale exceeds the store's build radius scale");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    check_lengths(ps);
    upload(D, ps, box, true, false);
    if (req.kind == 1) D.check(sfcnl_cu_set_sorted_field(D.ctx, "m", ps.field("m").data()));
    if (req.kind == 3) D.check(sfcnl_cu_set_sorted_field(D.ctx, "q", ps.field("q").data()));
    const sfcnl_build_params p = to_params(store.build);
    const std::uint8_t dummy = 0;
    D.check(sfcnl_cu_set_store(D.ctx, &p, store.n, store.counts.size(), store.counts.data(), store.offsets.data(),
                               store.blob.empty() ? &dummy : store.blob.data(), store.blob.size()));
    const int no = req.kind >= 2 ? 4 : 1;
    outputs.assign(no, std::vector<double>(n));
    neighbor_count.assign(n, 0);
    double* outs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int o = 0; o < no; ++o) outs[o] = outputs[o].data();
    const sfcnl_pass_params pp{req.kind, req.precision, req.query_scale, req.epsilon, req.sigma, req.coulomb_k};
    D.check(sfcnl_cu_reduce(D.ctx, &pp, outs, neighbor_count.data()));
}

void gpu::with_device_pass(const ParticleSet& ps, const SimulationBox& box, const NeighborStore& store,
                           const std::vector<std::string>& fields, const PassConfig& cfg,
                           const std::function<void(const sfcnl_cu_device_view&, const std::vector<const double*>&)>& fn) {
    const std::size_t n = ps.size();
    if (store.n != n) throw InputError("reduce: store/particle-set size mismatch");
    if (cfg.query_scale > store.build.build_radius_scale)
        throw InputError("reduce: query_scale exceeds the store's build radius scale");
    if (store.build.mode != ListMode::gather)
        throw InputError("reduce: user pair kernels on the GPU take gather stores");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    check_lengths(ps);
    upload(D, ps, box, true, false);
    std::vector<const double*> fp;
    for (const auto& name : fields) {
        D.check(sfcnl_cu_set_sorted_field(D.ctx, name.c_str(), ps.field(name).data()));
        const double* d = nullptr;
        D.check(sfcnl_cu_sorted_field_ptr(D.ctx, name.c_str(), &d));
        fp.push_back(d);
    }
    const sfcnl_build_params p = to_params(store.build);
    const std::uint8_t dummy = 0;
    D.check(sfcnl_cu_set_store(D.ctx, &p, store.n, store.counts.size(), store.counts.data(), store.offsets.data(),
                               store.blob.empty() ? &dummy : store.blob.data(), store.blob.size()));
    sfcnl_cu_device_view v{};
    D.check(sfcnl_cu_get_device_view(D.ctx, &v));
    fn(v, fp);
}

// ------------------------------------------------------------------ full Verlet list
FullVerletList build_full_list(const ParticleSet& ps, const SimulationBox& box, double build_scale, ListMode mode,
                               FullListMethod /*method*/, std::size_t /*cap*/) {
    if (mode != ListMode::gather) throw InputError("build_full_list: only gather lists are built on the GPU");
    if (!(build_scale >= 0)) throw InputError("build_full_list: build_scale must be >= 0");
    check_lengths(ps);
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const std::size_t n = ps.size();
    upload(D, ps, box, false, false);
    D.check(sfcnl_cu_sort_by_sfc(D.ctx, kDefaultSfcBits));
    D.check(sfcnl_cu_apply_order(D.ctx));
    std::uint64_t nn = 0, nsc = 0, nb = 0, pairs = 0;
    D.check(sfcnl_cu_build_octree(D.ctx, 64, &nn));
    sfcnl_build_params p{8, 8, 32, 0, 1, build_scale};
    D.check(sfcnl_cu_build_store(D.ctx, &p, &nsc, &nb));
    D.check(sfcnl_cu_build_full_list(D.ctx, build_scale, &pairs));
    FullVerletList sl;
    sl.mode = ListMode::gather;
    sl.build_scale = build_scale;
    sl.offsets.resize(n + 1);
    sl.neighbors.resize(pairs);
    D.check(sfcnl_cu_get_full_list(D.ctx, sl.offsets.data(), sl.neighbors.data()));
    std::vector<std::uint64_t> keys(n);
    std::vector<std::uint32_t> perm(n);
    D.check(sfcnl_cu_get_order(D.ctx, keys.data(), perm.data()));
    bool identity = true;
    for (std::size_t k = 0; k < n && identity; ++k) identity = perm[k] == k;
    if (identity) return sl;
    // sorted-index list -> the caller's numbering: row perm[s] holds perm[neighbors of s], ascending
    FullVerletList out;
    out.mode = ListMode::gather;
    out.build_scale = build_scale;
    out.offsets.assign(n + 1, 0);
    for (std::size_t s = 0; s < n; ++s) out.offsets[perm[s] + 1] = sl.offsets[s + 1] - sl.offsets[s];
    for (std::size_t i = 0; i < n; ++i) out.offsets[i + 1] += out.offsets[i];
    out.neighbors.resize(pairs);
    for (std::size_t s = 0; s < n; ++s) {
        std::uint32_t* row = out.neighbors.data() + out.offsets[perm[s]];
        const std::uint64_t b = sl.offsets[s], e = sl.offsets[s + 1];
        for (std::uint64_t k = b; k < e; ++k) row[k - b] = perm[sl.neighbors[k]];
        std::sort(row, row + (e - b));
    }
    return out;
}

void gpu::run_pass_full(const ParticleSet& ps, const SimulationBox& box, const FullVerletList& list,
                        const PassRequest& req, std::vector<std::vector<double>>& outputs,
                        std::vector<std::uint32_t>& neighbor_count) {
    const std::size_t n = ps.size();
    if (list.offsets.size() != n + 1) throw InputError("reduce_full: list/particle-set mismatch");
    if (req.query_scale > list.build_scale) throw InputError("reduce_full: query_scale exceeds the list's build scale");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    check_lengths(ps);
    upload(D, ps, box, true, false);
    if (req.kind == 1) D.check(sfcnl_cu_set_sorted_field(D.ctx, "m", ps.field("m").data()));
    if (req.kind == 3) D.check(sfcnl_cu_set_sorted_field(D.ctx, "q", ps.field("q").data()));
    const std::uint32_t dummy = 0;
    D.check(sfcnl_cu_set_full_list(D.ctx, n, list.mode == ListMode::symmetric ? 1 : 0, list.build_scale,
                                   list.offsets.data(), list.neighbors.empty() ? &dummy : list.neighbors.data(),
                                   list.neighbors.size()));
    const int no = req.kind >= 2 ? 4 : 1;
    outputs.assign(no, std::vector<double>(n));
    neighbor_count.assign(n, 0);
    double* outs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int o = 0; o < no; ++o) outs[o] = outputs[o].data();
    const sfcnl_pass_params pp{req.kind, req.precision, req.query_scale, req.epsilon, req.sigma, req.coulomb_k};
    D.check(sfcnl_cu_reduce_full(D.ctx, &pp, outs, neighbor_count.data()));
}

double bench::cluster_overhead(const NeighborStore& store, std::uint64_t true_directed_pairs) {
    if (store.build.mode != ListMode::gather) throw InputError("cluster_overhead: requires a gather-mode store");
    if (true_directed_pairs == 0) throw InputError("cluster_overhead: no in-range pairs");
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const sfcnl_build_params p = to_params(store.build);
    const std::uint8_t dummy = 0;
    D.check(sfcnl_cu_set_store(D.ctx, &p, store.n, store.counts.size(), store.counts.data(), store.offsets.data(),
                               store.blob.empty() ? &dummy : store.blob.data(), store.blob.size()));
    std::uint64_t slots = 0;
    D.check(sfcnl_cu_cluster_slots(D.ctx, &slots));
    return double(slots) / double(true_directed_pairs);
}

// ------------------------------------------------------------------ store helpers
std::uint64_t entry_mask(const std::uint8_t* rec, std::uint32_t entry, std::uint32_t mask_bytes) {
    std::uint64_t m = 0;
    for (std::uint32_t b = 0; b < mask_bytes; ++b) m |= std::uint64_t(rec[std::size_t(entry) * mask_bytes + b]) << (8 * b);
    return m;
}

const std::uint8_t* decode_entry_indices(const NeighborStore& store, std::uint64_t sc, std::uint32_t* out) {
    if (sc >= store.num_superclusters()) throw InputError("decode_entry_indices: super-cluster out of range");
    const std::uint32_t count = store.counts[sc];
    const std::uint64_t begin = store.offsets[sc], end = store.offsets[sc + 1];
    const std::uint64_t mb = std::uint64_t(count) * store.build.params.mask_bytes_per_entry();
    if (begin + mb > end) throw DecodeError("blob slice too short for bitmasks", std::size_t(begin));
    const std::uint8_t* rec = store.blob.data() + begin;
    const std::uint64_t len = end - begin - mb;
    if (store.build.compress) {
        const std::size_t used = codec::decode_into(rec + mb, std::size_t(len), count, store.build.params.w, out);
        if (used != len) throw DecodeError("trailing bytes in index blob", used);
    } else {
        if (len != std::uint64_t(count) * 4) throw DecodeError("raw index blob length mismatch", std::size_t(len));
        if (count) std::memcpy(out, rec + mb, std::size_t(count) * 4);
    }
    return rec;
}

std::vector<NeighborEntry> neighbor_clusters(const NeighborStore& store, std::uint64_t sc) {
    const std::uint32_t count = store.counts.at(sc);
    std::vector<std::uint32_t> idx(count);
    const std::uint8_t* rec = decode_entry_indices(store, sc, idx.data());
    std::vector<NeighborEntry> out(count);
    for (std::uint32_t e = 0; e < count; ++e) out[e] = {idx[e], entry_mask(rec, e, store.build.params.mask_bytes_per_entry())};
    return out;
}

MemoryFootprint memory_footprint(const NeighborStore& s) {
    MemoryFootprint f;
    f.total_bytes = s.total_bytes();
    f.bytes_per_particle = s.n ? double(f.total_bytes) / double(s.n) : 0.0;
    return f;
}

namespace {
const char kMagic[8] = {'S', 'F', 'N', 'L', 'S', 'T', 'O', 'R'};
template <class T>
void put(std::ostream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof v);
}
template <class T>
T get(std::istream& i) {
    T v{};
    i.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!i) throw DecodeError("store file truncated", std::size_t(i.tellg()));
    return v;
}
}  // namespace

void write_store(const NeighborStore& s, std::ostream& out) {
    out.write(kMagic, 8);
    put<std::uint32_t>(out, 1);
    put<std::uint8_t>(out, std::uint8_t(s.build.mode));
    put<std::uint8_t>(out, s.build.compress ? 1 : 0);
    put<std::uint16_t>(out, 0);
    put<std::uint32_t>(out, s.build.params.ci);
    put<std::uint32_t>(out, s.build.params.cj);
    put<std::uint32_t>(out, s.build.params.sc_size);
    put<std::uint32_t>(out, std::uint32_t(s.build.params.w));
    put<double>(out, s.build.build_radius_scale);
    put<std::uint64_t>(out, s.n);
    put<std::uint64_t>(out, s.counts.size());
    put<std::uint64_t>(out, s.blob.size());
    out.write(reinterpret_cast<const char*>(s.counts.data()), std::streamsize(s.counts.size() * 4));
    out.write(reinterpret_cast<const char*>(s.offsets.data()), std::streamsize(s.offsets.size() * 8));
    out.write(reinterpret_cast<const char*>(s.blob.data()), std::streamsize(s.blob.size()));
    if (!out) throw std::runtime_error("write_store: stream failure");
}

void write_store(const NeighborStore& s, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("write_store: cannot open " + path);
    write_store(s, f);
}

NeighborStore read_store(std::istream& in) {
    char magic[8];
    in.read(magic, 8);
    if (!in || std::memcmp(magic, kMagic, 8) != 0) throw DecodeError("bad store magic", 0);
    if (get<std::uint32_t>(in) != 1) throw DecodeError("unsupported store version", 8);
    const auto mode = get<std::uint8_t>(in);
    const auto comp = get<std::uint8_t>(in);
    (void)get<std::uint16_t>(in);
    const auto ci = get<std::uint32_t>(in), cj = get<std::uint32_t>(in), scs = get<std::uint32_t>(in);
    const auto w = get<std::uint32_t>(in);
    if (scs != kSuperClusterSize) throw DecodeError("unsupported super-cluster size", 0);
    const auto scale = get<double>(in);
    NeighborStore s;
    s.build = BuildParams(ClusterParams(ci, cj, int(w)), mode == 0 ? ListMode::gather : ListMode::symmetric, comp != 0, scale);
    s.n = get<std::uint64_t>(in);
    const auto nsc = get<std::uint64_t>(in), nb = get<std::uint64_t>(in);
    s.counts.resize(nsc);
    s.offsets.resize(nsc + 1);
    s.blob.resize(nb);
    in.read(reinterpret_cast<char*>(s.counts.data()), std::streamsize(nsc * 4));
    in.read(reinterpret_cast<char*>(s.offsets.data()), std::streamsize((nsc + 1) * 8));
    in.read(reinterpret_cast<char*>(s.blob.data()), std::streamsize(nb));
    if (!in) throw DecodeError("store file truncated", std::size_t(in.tellg()));
    return s;
}

NeighborStore read_store(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("read_store: cannot open " + path);
    return read_store(f);
}

// ------------------------------------------------------------------ codec (host)
namespace codec {

std::vector<std::uint64_t> delta_encode(std::span<const std::uint32_t> idx) {
    std::vector<std::uint64_t> d(idx.size());
    for (std::size_t k = 0; k < idx.size(); ++k) {
        if (k && idx[k] <= idx[k - 1]) throw InputError("delta_encode: input not strictly increasing");
        d[k] = k ? std::uint64_t(idx[k]) - idx[k - 1] : std::uint64_t(idx[0]) + 1;
    }
    return d;
}

static int nibbles_of(std::uint64_t v) {
    int b = 0;
    while (v) ++b, v >>= 1;
    return (b + 3) / 4;
}

EncodedBlock encode_block(std::span<const std::uint64_t> diffs, int w) {
    check_block_width(w);
    if (diffs.size() > std::size_t(w)) throw InputError("encode_block: more differences than block width");
    EncodedBlock b;
    for (std::size_t k = 0; k < diffs.size(); ++k) {
        const std::uint64_t v = diffs[k];
        if (v == 0) throw InputError("encode_block: difference of zero");
        if (v > 0xffffffffull) throw InputError("encode_block: difference exceeds 2^32 - 1");
        if (v == 1) continue;
        b.bitmask |= std::uint64_t(1) << k;
        if (v <= 9) {
            b.info_nibbles.push_back(std::uint8_t(v + 6));
            continue;
        }
        const int nn = nibbles_of(v);
        b.info_nibbles.push_back(std::uint8_t(nn - 1));
        for (int p = nn - 1; p >= 0; --p) b.data_nibbles.push_back(std::uint8_t((v >> (4 * p)) & 15u));
    }
    return b;
}

std::vector<std::uint64_t> decode_block(const EncodedBlock& b, std::size_t len) {
    std::vector<std::uint64_t> d(len, 1);
    std::size_t ii = 0, di = 0;
    for (std::size_t k = 0; k < len; ++k) {
        if (!((b.bitmask >> k) & 1u)) continue;
        if (ii >= b.info_nibbles.size()) throw DecodeError("missing info nibble", 0);
        const std::uint8_t nib = b.info_nibbles[ii++];
        if (nib >= 8) {
            d[k] = std::uint64_t(nib) - 6;
            continue;
        }
        std::uint64_t v = 0;
        for (int p = 0; p <= nib; ++p) {
            if (di >= b.data_nibbles.size()) throw DecodeError("missing data nibble", 0);
            v = (v << 4) | b.data_nibbles[di++];
        }
        d[k] = v;
    }
    return d;
}

EncodedList encode(std::span<const std::uint32_t> idx, int w) {
    check_block_width(w);
    EncodedList e;
    e.count = std::uint32_t(idx.size());
    std::uint64_t len = 0;
    host_check(sfcnl_codec_encode(idx.data(), idx.size(), w, nullptr, 0, &len));
    e.bytes.resize(len);
    if (len) host_check(sfcnl_codec_encode(idx.data(), idx.size(), w, e.bytes.data(), len, &len));
    return e;
}

std::size_t decode_into(const std::uint8_t* data, std::size_t size, std::uint32_t count, int w, std::uint32_t* out) {
    check_block_width(w);
    std::uint64_t used = 0;
    static const std::uint8_t none = 0;
    host_check(sfcnl_codec_decode_into(size ? data : &none, size, count, w, out, &used));
    return std::size_t(used);
}

std::vector<std::uint32_t> decode(const EncodedList& list, int w) {
    std::vector<std::uint32_t> out(list.count);
    const std::size_t used = decode_into(list.bytes.data(), list.bytes.size(), list.count, w, out.data());
    if (used != list.bytes.size()) throw DecodeError("trailing bytes after encoded list", used);
    return out;
}

int encoded_size_bits(std::uint64_t v) {
    if (v == 0) throw InputError("encoded_size_bits: zero difference");
    if (v > 0xffffffffull) throw InputError("encoded_size_bits: difference exceeds 2^32 - 1");
    return v == 1 ? 1 : (v <= 9 ? 5 : 5 + 4 * nibbles_of(v));
}

int size_stream_vbyte(std::uint64_t v) {
    if (v >= (std::uint64_t(1) << 32)) throw InputError("size_stream_vbyte: value exceeds 32 bits");
    return v < (1u << 8) ? 10 : (v < (1u << 16) ? 18 : (v < (1u << 24) ? 26 : 34));
}

int size_band(std::uint64_t v) {
    if (v == 0 || v > (std::uint64_t(1) << 32)) throw InputError("size_band: value out of range [1, 2^32]");
    return v <= 2 ? 2 : (v <= 256 ? 10 : 34);
}

}  // namespace codec

// ------------------------------------------------------------------ generators
static ParticleSet generated(std::size_t n, std::vector<double> (&a)[6], const double* box6, SimulationBox& box,
                             std::array<bool, 3> per) {
    ParticleSet ps;
    ps.x = std::move(a[0]), ps.y = std::move(a[1]), ps.z = std::move(a[2]), ps.h = std::move(a[3]);
    ps.fields.emplace("m", std::move(a[4]));
    ps.fields.emplace("q", std::move(a[5]));
    box = SimulationBox({box6[0], box6[1], box6[2]}, {box6[3], box6[4], box6[5]}, per);
    (void)n;
    return ps;
}

ParticleSet make_uniform(const UniformSpec& s, SimulationBox& box) {
    std::vector<double> a[6];
    for (auto& v : a) v.resize(s.n);
    double box6[6];
    const std::int32_t per[3] = {s.periodic[0], s.periodic[1], s.periodic[2]};
    host_check(sfcnl_make_uniform(s.n, s.density, s.target_neighbors, per, s.h_jitter, s.seed, a[0].data(), a[1].data(),
                                  a[2].data(), a[3].data(), a[4].data(), a[5].data(), box6));
    return generated(s.n, a, box6, box, s.periodic);
}

ParticleSet make_evrard(const EvrardSpec& s, SimulationBox& box) {
    std::vector<double> a[6];
    for (auto& v : a) v.resize(s.n);
    double box6[6];
    const std::int32_t per[3] = {s.periodic[0], s.periodic[1], s.periodic[2]};
    host_check(sfcnl_make_evrard(s.n, s.target_neighbors, s.constant_h ? 1 : 0, per, s.seed, a[0].data(), a[1].data(),
                                 a[2].data(), a[3].data(), a[4].data(), a[5].data(), box6));
    return generated(s.n, a, box6, box, s.periodic);
}

double uniform_h_for_target(double target, double rho) {
    if (!(target > 0) || !(rho > 0)) throw InputError("uniform_h_for_target: positive inputs required");
    return std::cbrt(3.0 * target / (4.0 * std::numbers::pi_v<double> * rho));
}

// ------------------------------------------------------------------ ISA (compatibility)
bool cpu_supports_avx2() {
#if defined(__x86_64__)
    return __builtin_cpu_supports("avx2");
#else
    return false;
#endif
}
bool compiled_with_avx2() { return false; }
Isa resolve_isa(Isa requested) {
    if (requested == Isa::avx2) throw InputError("AVX2 support not compiled in (B200 build: the pass runs on the GPU)");
    return Isa::scalar;
}
const char* isa_name(Isa isa) { return isa == Isa::automatic ? "auto" : (isa == Isa::scalar ? "scalar" : "avx2"); }

}  // namespace sfcnl
