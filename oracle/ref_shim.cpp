// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference C++ library, compiled from the
// reference's own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libsfcnl_ref.so (git-ignored; it travels to the GPU box). The
// reference namespace is renamed at compile time (-Dsfcnl=sfcnl_ref) so this
// library can share a process with the B200 drop-in, which owns `sfcnl::`.
//
// Every entry point forwards to the reference API it names:
//   ref_make_uniform / ref_make_evrard   generators.hpp:34-35, generators.cpp:21-82
//   ref_sort_by_sfc                      hilbert.hpp:126, hilbert.cpp:8-26
//   ref_hilbert_encode / _decode         hilbert.hpp:66-90
//   ref_build_octree / ref_octree_*      octree.hpp:51-60, octree.cpp:43-96
//   ref_build_store / ref_store_*        neighbor_build.hpp:18-19, neighbor_build.cpp:74-184
//   ref_reduce                           reduce.hpp:38-231 (+ simd_avx2.cpp when isa=avx2)
//   ref_codec_*                          nibble_codec.hpp:20-63
//   ref_pipeline                         the run_bench sequence (bench.cpp:147-186), all stages timed
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sfcnl/baselines.hpp"
#include "sfcnl/bench.hpp"
#include "sfcnl/builtin_kernels.hpp"
#include "sfcnl/generators.hpp"
#include "sfcnl/hilbert.hpp"
#include "sfcnl/neighbor_build.hpp"
#include "sfcnl/nibble_codec.hpp"
#include "sfcnl/octree.hpp"
#include "sfcnl/reduce.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;
thread_local uint64_t g_err_off = 0;

// 0 ok, 1 InputError, 2 BuildError, 3 DecodeError, 4 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sfcnl_ref::DecodeError& e) {
        g_err = e.what();
        g_err_off = e.byte_offset;
        return 3;
    } catch (const sfcnl_ref::InputError& e) {
        g_err = e.what();
        return 1;
    } catch (const sfcnl_ref::BuildError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

sfcnl_ref::SimulationBox make_box(const double* box6, const int* per) {
    return sfcnl_ref::SimulationBox({box6[0], box6[1], box6[2]}, {box6[3], box6[4], box6[5]},
                                    {per[0] != 0, per[1] != 0, per[2] != 0});
}

sfcnl_ref::ParticleSet make_ps(uint64_t n, const double* x, const double* y, const double* z,
                               const double* h, const double* m, const double* q) {
    sfcnl_ref::ParticleSet ps;
    ps.x.assign(x, x + n);
    ps.y.assign(y, y + n);
    ps.z.assign(z, z + n);
    ps.h.assign(h, h + n);
    if (m) ps.fields.emplace("m", std::vector<double>(m, m + n));
    if (q) ps.fields.emplace("q", std::vector<double>(q, q + n));
    return ps;
}

void export_ps(const sfcnl_ref::ParticleSet& ps, double* x, double* y, double* z, double* h,
               double* m, double* q) {
    const size_t n = ps.size();
    std::memcpy(x, ps.x.data(), n * 8);
    std::memcpy(y, ps.y.data(), n * 8);
    std::memcpy(z, ps.z.data(), n * 8);
    std::memcpy(h, ps.h.data(), n * 8);
    if (m) std::memcpy(m, ps.field("m").data(), n * 8);
    if (q) std::memcpy(q, ps.field("q").data(), n * 8);
}

sfcnl_ref::NeighborStore make_store(uint64_t n, uint32_t ci, uint32_t cj, int w, int mode,
                                    int compress, double scale, uint64_t num_sc,
                                    const uint32_t* counts, const uint64_t* offsets,
                                    const uint8_t* blob, uint64_t blob_size) {
    sfcnl_ref::NeighborStore s;
    s.build = sfcnl_ref::BuildParams(sfcnl_ref::ClusterParams(ci, cj, w),
                                     mode ? sfcnl_ref::ListMode::symmetric
                                          : sfcnl_ref::ListMode::gather,
                                     compress != 0, scale);
    s.n = n;
    s.counts.assign(counts, counts + num_sc);
    s.offsets.assign(offsets, offsets + num_sc + 1);
    s.blob.assign(blob, blob + blob_size);
    return s;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

REF_API const char* ref_last_error(uint64_t* byte_offset) {
    if (byte_offset) *byte_offset = g_err_off;
    return g_err.c_str();
}

REF_API int ref_make_uniform(uint64_t n, double density, double target, const int* per,
                             double h_jitter, uint64_t seed, double* x, double* y, double* z,
                             double* h, double* m, double* q, double* box6) {
    return guarded([&] {
        sfcnl_ref::UniformSpec s;
        s.n = n;
        s.density = density;
        s.target_neighbors = target;
        s.periodic = {per[0] != 0, per[1] != 0, per[2] != 0};
        s.h_jitter = h_jitter;
        s.seed = seed;
        sfcnl_ref::SimulationBox box;
        const auto ps = sfcnl_ref::make_uniform(s, box);
        export_ps(ps, x, y, z, h, m, q);
        for (int d = 0; d < 3; ++d) box6[d] = box.lo[d], box6[3 + d] = box.hi[d];
    });
}

REF_API int ref_make_evrard(uint64_t n, double target, int constant_h, const int* per,
                            uint64_t seed, double* x, double* y, double* z, double* h, double* m,
                            double* q, double* box6) {
    return guarded([&] {
        sfcnl_ref::EvrardSpec s;
        s.n = n;
        s.target_neighbors = target;
        s.constant_h = constant_h != 0;
        s.periodic = {per[0] != 0, per[1] != 0, per[2] != 0};
        s.seed = seed;
        sfcnl_ref::SimulationBox box;
        const auto ps = sfcnl_ref::make_evrard(s, box);
        export_ps(ps, x, y, z, h, m, q);
        for (int d = 0; d < 3; ++d) box6[d] = box.lo[d], box6[3 + d] = box.hi[d];
    });
}

REF_API int ref_hilbert_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint64_t* key) {
    return guarded([&] { *key = sfcnl_ref::hilbert_encode(ix, iy, iz, bits); });
}

REF_API int ref_hilbert_decode(uint64_t key, int bits, uint32_t* xyz) {
    return guarded([&] {
        const auto a = sfcnl_ref::hilbert_decode(key, bits);
        xyz[0] = a[0], xyz[1] = a[1], xyz[2] = a[2];
    });
}

REF_API int ref_sfc_key(double x, double y, double z, const double* box6, const int* per,
                        int bits, uint64_t* key) {
    return guarded([&] { *key = sfcnl_ref::sfc_key({x, y, z}, make_box(box6, per), bits); });
}

REF_API int ref_sort_by_sfc(uint64_t n, const double* x, const double* y, const double* z,
                            const double* h, const double* box6, const int* per, int bits,
                            uint64_t* keys, uint32_t* perm) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const auto o = sfcnl_ref::sort_by_sfc(ps, make_box(box6, per), bits);
        std::memcpy(keys, o.keys.data(), n * 8);
        std::memcpy(perm, o.perm.data(), n * 4);
    });
}

// ---- octree -----------------------------------------------------------------
struct RefTree {
    sfcnl_ref::Octree t;
};

REF_API int ref_build_octree(uint64_t n, const uint64_t* keys, int bits, uint32_t bucket,
                             void** out) {
    return guarded([&] {
        sfcnl_ref::SfcOrder o;
        o.bits = bits;
        o.keys.assign(keys, keys + n);
        o.perm.resize(n);
        auto* t = new RefTree{sfcnl_ref::build_octree(o, bucket)};
        *out = t;
    });
}

REF_API uint64_t ref_octree_size(void* h) { return static_cast<RefTree*>(h)->t.nodes.size(); }

// Node record layout (matches OctreeNode field order, octree.hpp:11-21).
REF_API void ref_octree_nodes(void* h, uint64_t* key_first, uint64_t* key_last,
                              uint32_t* pbegin, uint32_t* pend, int32_t* first_child,
                              uint8_t* depth) {
    const auto& nodes = static_cast<RefTree*>(h)->t.nodes;
    for (size_t k = 0; k < nodes.size(); ++k) {
        key_first[k] = nodes[k].key_first;
        key_last[k] = nodes[k].key_last;
        pbegin[k] = nodes[k].particle_begin;
        pend[k] = nodes[k].particle_end;
        first_child[k] = nodes[k].first_child;
        depth[k] = nodes[k].depth;
    }
}

REF_API void ref_octree_free(void* h) { delete static_cast<RefTree*>(h); }

static sfcnl_ref::Octree tree_from_arrays(uint64_t n, int bits, uint64_t num_nodes,
                                          const uint64_t* key_first, const uint64_t* key_last,
                                          const uint32_t* pbegin, const uint32_t* pend,
                                          const int32_t* first_child, const uint8_t* depth) {
    sfcnl_ref::Octree t;
    t.bits = bits;
    t.n = uint32_t(n);
    t.nodes.resize(num_nodes);
    for (uint64_t k = 0; k < num_nodes; ++k) {
        t.nodes[k].key_first = key_first[k];
        t.nodes[k].key_last = key_last[k];
        t.nodes[k].particle_begin = pbegin[k];
        t.nodes[k].particle_end = pend[k];
        t.nodes[k].first_child = first_child[k];
        t.nodes[k].depth = depth[k];
    }
    return t;
}

// lo/hi: [num_nodes * 3] each (x,y,z interleaved per node); radius: [num_nodes].
REF_API int ref_node_geometry(void* tree, uint64_t n, const double* x, const double* y,
                              const double* z, const double* h, double* lo, double* hi,
                              double* radius) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const auto& t = static_cast<RefTree*>(tree)->t;
        const auto boxes = sfcnl_ref::compute_node_aabbs(t, ps);
        const auto rad = sfcnl_ref::compute_node_max_radius(t, ps);
        for (size_t k = 0; k < boxes.size(); ++k) {
            for (int d = 0; d < 3; ++d) {
                lo[3 * k + d] = boxes[k].lo[d];
                hi[3 * k + d] = boxes[k].hi[d];
            }
            radius[k] = rad[k];
        }
    });
}

// ---- neighbor store -----------------------------------------------------------
struct RefStore {
    sfcnl_ref::NeighborStore s;
};

REF_API int ref_build_store(uint64_t n, const double* x, const double* y, const double* z,
                            const double* h, const double* box6, const int* per, void* tree,
                            uint32_t ci, uint32_t cj, int w, int mode, int compress,
                            double scale, int threads, void** out) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const sfcnl_ref::BuildParams bp(
            sfcnl_ref::ClusterParams(ci, cj, w),
            mode ? sfcnl_ref::ListMode::symmetric : sfcnl_ref::ListMode::gather, compress != 0,
            scale);
        auto* s = new RefStore{sfcnl_ref::build_neighbor_store(
            ps, make_box(box6, per), static_cast<RefTree*>(tree)->t, bp, threads)};
        *out = s;
    });
}

// Same, with the tree given as node arrays (so a GPU-built tree can be fed in).
REF_API int ref_build_store_nodes(uint64_t n, const double* x, const double* y, const double* z,
                                  const double* h, const double* box6, const int* per, int bits,
                                  uint64_t num_nodes, const uint64_t* key_first,
                                  const uint64_t* key_last, const uint32_t* pbegin,
                                  const uint32_t* pend, const int32_t* first_child,
                                  const uint8_t* depth, uint32_t ci, uint32_t cj, int w,
                                  int mode, int compress, double scale, int threads, void** out) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const auto t = tree_from_arrays(n, bits, num_nodes, key_first, key_last, pbegin, pend,
                                        first_child, depth);
        const sfcnl_ref::BuildParams bp(
            sfcnl_ref::ClusterParams(ci, cj, w),
            mode ? sfcnl_ref::ListMode::symmetric : sfcnl_ref::ListMode::gather, compress != 0,
            scale);
        *out = new RefStore{sfcnl_ref::build_neighbor_store(ps, make_box(box6, per), t, bp, threads)};
    });
}

// write_store (neighbor_store.cpp:84-103) of a built store to `path` (SFNLSTOR v1).
REF_API int ref_store_write(void* h, const char* path) {
    return guarded([&] { sfcnl_ref::write_store(static_cast<RefStore*>(h)->s, std::string(path)); });
}

REF_API void ref_store_info(void* h, uint64_t* num_sc, uint64_t* blob_size) {
    const auto& s = static_cast<RefStore*>(h)->s;
    *num_sc = s.counts.size();
    *blob_size = s.blob.size();
}

REF_API void ref_store_copy(void* h, uint32_t* counts, uint64_t* offsets, uint8_t* blob) {
    const auto& s = static_cast<RefStore*>(h)->s;
    std::memcpy(counts, s.counts.data(), s.counts.size() * 4);
    std::memcpy(offsets, s.offsets.data(), s.offsets.size() * 8);
    if (!s.blob.empty()) std::memcpy(blob, s.blob.data(), s.blob.size());
}

REF_API void ref_store_free(void* h) { delete static_cast<RefStore*>(h); }

// ---- neighborhood pass --------------------------------------------------------
// kernel: 0 count, 1 density, 2 lj, 3 lj+coulomb. real: 0 double, 1 float.
// isa: 0 auto, 1 scalar, 2 avx2. outs: num_outputs arrays of n (double; float results widened).
REF_API int ref_reduce(int kernel, int real, uint64_t n, const double* x, const double* y,
                       const double* z, const double* h, const double* m, const double* q,
                       const double* box6, const int* per, uint32_t ci, uint32_t cj, int w,
                       int mode, int compress, double scale, uint64_t num_sc,
                       const uint32_t* counts, const uint64_t* offsets, const uint8_t* blob,
                       uint64_t blob_size, double query_scale, int isa, int threads, double eps,
                       double sigma, double ck, double** outs, uint32_t* ncount) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, m, q);
        const auto box = make_box(box6, per);
        const auto store = make_store(n, ci, cj, w, mode, compress, scale, num_sc, counts,
                                      offsets, blob, blob_size);
        const sfcnl_ref::PassConfig cfg(query_scale, sfcnl_ref::Isa(isa), threads);
        auto run = [&](auto real_tag) {
            using Real = decltype(real_tag);
            auto finish = [&](const sfcnl_ref::ReduceResult<Real>& r) {
                for (size_t o = 0; o < r.outputs.size(); ++o)
                    for (uint64_t i = 0; i < n; ++i) outs[o][i] = double(r.outputs[o][i]);
                std::memcpy(ncount, r.neighbor_count.data(), n * 4);
            };
            switch (kernel) {
                case 0: finish(sfcnl_ref::reduce<Real>(ps, box, store, sfcnl_ref::count_kernel<Real>(), cfg)); break;
                case 1: finish(sfcnl_ref::reduce<Real>(ps, box, store, sfcnl_ref::sph_density_kernel<Real>(), cfg)); break;
                case 2: finish(sfcnl_ref::reduce<Real>(ps, box, store, sfcnl_ref::lj_kernel<Real>(Real(eps), Real(sigma)), cfg)); break;
                case 3: finish(sfcnl_ref::reduce<Real>(ps, box, store, sfcnl_ref::lj_coulomb_kernel<Real>(Real(eps), Real(sigma), Real(ck)), cfg)); break;
                default: throw sfcnl_ref::InputError("ref_reduce: unknown kernel id");
            }
        };
        if (real) run(float{}); else run(double{});
    });
}

// ---- full Verlet list baseline (baselines.hpp:39-131) ----------------------------
struct RefFull {
    sfcnl_ref::FullVerletList l;
};

REF_API int ref_full_list(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                          const double* box6, const int* per, double build_scale, int mode, int method,
                          void** out, uint64_t* num_pairs) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        auto* r = new RefFull{sfcnl_ref::build_full_list(
            ps, make_box(box6, per), build_scale, mode ? sfcnl_ref::ListMode::symmetric : sfcnl_ref::ListMode::gather,
            sfcnl_ref::FullListMethod(method), ~size_t(0))};
        *num_pairs = r->l.neighbors.size();
        *out = r;
    });
}

REF_API void ref_full_copy(void* h, uint64_t* offsets, uint32_t* neighbors) {
    const auto& l = static_cast<RefFull*>(h)->l;
    std::memcpy(offsets, l.offsets.data(), l.offsets.size() * 8);
    if (!l.neighbors.empty()) std::memcpy(neighbors, l.neighbors.data(), l.neighbors.size() * 4);
}

REF_API int ref_reduce_full(void* hl, int kernel, uint64_t n, const double* x, const double* y, const double* z,
                            const double* h, const double* m, const double* q, const double* box6, const int* per,
                            double query_scale, double eps, double sigma, double ck, double** outs,
                            uint32_t* ncount) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, m, q);
        const auto box = make_box(box6, per);
        const auto& l = static_cast<RefFull*>(hl)->l;
        const sfcnl_ref::PassConfig cfg(query_scale, sfcnl_ref::Isa::scalar, 1);
        auto finish = [&](const sfcnl_ref::ReduceResult<double>& r) {
            for (size_t o = 0; o < r.outputs.size(); ++o)
                for (uint64_t i = 0; i < n; ++i) outs[o][i] = r.outputs[o][i];
            std::memcpy(ncount, r.neighbor_count.data(), n * 4);
        };
        switch (kernel) {
            case 0: finish(sfcnl_ref::reduce_full<double>(ps, box, l, sfcnl_ref::count_kernel<double>(), cfg)); break;
            case 1: finish(sfcnl_ref::reduce_full<double>(ps, box, l, sfcnl_ref::sph_density_kernel<double>(), cfg)); break;
            case 2: finish(sfcnl_ref::reduce_full<double>(ps, box, l, sfcnl_ref::lj_kernel<double>(eps, sigma), cfg)); break;
            default: throw sfcnl_ref::InputError("ref_reduce_full: unknown kernel id");
        }
    });
}

REF_API void ref_full_free(void* h) { delete static_cast<RefFull*>(h); }

// ---- codec --------------------------------------------------------------------
REF_API int ref_codec_encode(const uint32_t* idx, uint64_t count, int w, uint8_t* out,
                             uint64_t cap, uint64_t* len) {
    return guarded([&] {
        const auto e = sfcnl_ref::codec::encode({idx, size_t(count)}, w);
        *len = e.bytes.size();
        if (e.bytes.size() <= cap && !e.bytes.empty()) std::memcpy(out, e.bytes.data(), e.bytes.size());
    });
}

REF_API int ref_codec_decode_into(const uint8_t* data, uint64_t size, uint32_t count, int w,
                                  uint32_t* out, uint64_t* consumed) {
    return guarded([&] { *consumed = sfcnl_ref::codec::decode_into(data, size, count, w, out); });
}

// ---- brute-force oracle ------------------------------------------------------
REF_API int ref_brute_force_counts(uint64_t n, const double* x, const double* y, const double* z,
                                   const double* h, const double* box6, const int* per,
                                   double scale, int mode, uint32_t* out) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const auto c = sfcnl_ref::brute_force_counts(
            ps, make_box(box6, per), scale,
            mode ? sfcnl_ref::ListMode::symmetric : sfcnl_ref::ListMode::gather, n + 1);
        std::memcpy(out, c.data(), n * 4);
    });
}

REF_API int ref_cluster_overhead(uint64_t n, uint32_t ci, uint32_t cj, int w, int compress,
                                 uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
                                 const uint8_t* blob, uint64_t blob_size, uint64_t true_pairs,
                                 double* out) {
    return guarded([&] {
        const auto s = make_store(n, ci, cj, w, 0, compress, 1.0, num_sc, counts, offsets, blob,
                                  blob_size);
        *out = sfcnl_ref::bench::cluster_overhead(s, true_pairs);
    });
}

// ---- full pipeline, every stage timed (CPU baseline) ---------------------------
// times_ms[7]: sort_by_sfc, apply_sfc_order, build_octree, build_neighbor_store,
//              reduce density, reduce lj, total. out_stats[4]: bytes/particle,
//              mean neighbours, entries, blob bytes.
REF_API int ref_pipeline(uint64_t n, const double* x, const double* y, const double* z,
                         const double* h, const double* m, const double* box6, const int* per,
                         uint32_t ci, uint32_t cj, int w, double scale, int threads, double eps,
                         double sigma, int do_lj, double* times_ms, double* out_stats,
                         double* rho_out) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, m, nullptr);
        const auto box = make_box(box6, per);
        const double t0 = now_ms();
        const auto order = sfcnl_ref::sort_by_sfc(ps, box);
        const double t1 = now_ms();
        const auto sorted = sfcnl_ref::apply_sfc_order(ps, order);
        const double t2 = now_ms();
        const auto tree = sfcnl_ref::build_octree(order, 64);
        const double t3 = now_ms();
        const sfcnl_ref::BuildParams bp(sfcnl_ref::ClusterParams(ci, cj, w),
                                        sfcnl_ref::ListMode::gather, true, scale);
        const auto store = sfcnl_ref::build_neighbor_store(sorted, box, tree, bp, threads);
        const double t4 = now_ms();
        const sfcnl_ref::PassConfig cfg(1.0, sfcnl_ref::Isa::automatic, threads);
        const auto dens = sfcnl_ref::reduce<double>(sorted, box, store,
                                                    sfcnl_ref::sph_density_kernel<double>(), cfg);
        const double t5 = now_ms();
        double t6 = t5;
        if (do_lj) {
            const auto lj = sfcnl_ref::reduce<double>(
                sorted, box, store, sfcnl_ref::lj_kernel<double>(eps, sigma), cfg);
            t6 = now_ms();
        }
        times_ms[0] = t1 - t0;
        times_ms[1] = t2 - t1;
        times_ms[2] = t3 - t2;
        times_ms[3] = t4 - t3;
        times_ms[4] = t5 - t4;
        times_ms[5] = t6 - t5;
        times_ms[6] = t6 - t0;
        uint64_t total = 0, entries = 0;
        for (auto c : dens.neighbor_count) total += c;
        for (auto c : store.counts) entries += c;
        out_stats[0] = sfcnl_ref::memory_footprint(store).bytes_per_particle;
        out_stats[1] = n ? double(total) / double(n) : 0.0;
        out_stats[2] = double(entries);
        out_stats[3] = double(store.blob.size());
        if (rho_out) std::memcpy(rho_out, dens.output("rho").data(), n * 8);
    });
}

// ---- per-cluster geometry (compute_cluster_geometry, neighbor_build.cpp:19-38) ---------
// Clusters [k*width, min((k+1)*width, n)) through the reference's own cluster_aabb /
// cluster_max_radius (cluster.hpp:77-90). lo/hi: [ncl*3], maxh: [ncl].
REF_API int ref_cluster_geometry(uint64_t n, const double* x, const double* y, const double* z,
                                 const double* h, uint32_t width, double* lo, double* hi,
                                 double* maxh) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const uint64_t ncl = (n + width - 1) / width;
        for (uint64_t k = 0; k < ncl; ++k) {
            const uint64_t b = k * width, e = std::min<uint64_t>(b + width, n);
            const auto a = sfcnl_ref::cluster_aabb(ps, b, e);
            for (int d = 0; d < 3; ++d) lo[3 * k + d] = a.lo[d], hi[3 * k + d] = a.hi[d];
            maxh[k] = sfcnl_ref::cluster_max_radius(ps, b, e);
        }
    });
}

// ---- LJ normwise tolerance denominators ------------------------------------------
// sum_j |F_ij| and sum_j |E_ij| over each particle's in-range neighbourhood, computed by
// the reference's own reduce<double> (reduce.hpp:38-231) with a user pair kernel built by
// make_pair_kernel (pair_kernel.hpp:81-91): the same pair set and term formulas as
// LjKernel (builtin_kernels.hpp:54-66), absolute values summed.
REF_API int ref_lj_abs_sums(uint64_t n, const double* x, const double* y, const double* z,
                            const double* h, const double* box6, const int* per, uint32_t ci,
                            uint32_t cj, int w, int mode, int compress, double scale,
                            uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
                            const uint8_t* blob, uint64_t blob_size, double query_scale,
                            int threads, double eps, double sigma, double* absf, double* abse) {
    return guarded([&] {
        const auto ps = make_ps(n, x, y, z, h, nullptr, nullptr);
        const auto box = make_box(box6, per);
        const auto store = make_store(n, ci, cj, w, mode, compress, scale, num_sc, counts,
                                      offsets, blob, blob_size);
        using sfcnl_ref::OutputSpec;
        auto k = sfcnl_ref::make_pair_kernel<double, 0, 2>(
            std::array<const char*, 0>{},
            std::array<OutputSpec, 2>{{{"absf", sfcnl_ref::Symmetry::even, sfcnl_ref::Reduction::sum},
                                       {"abse", sfcnl_ref::Symmetry::even, sfcnl_ref::Reduction::sum}}},
            [eps, sigma](const sfcnl_ref::PairArgs<double>& a, const std::array<double, 0>&,
                         const std::array<double, 0>&) -> std::array<double, 2> {
                const double inv2 = 1.0 / a.d2;
                const double s2 = sigma * sigma * inv2;
                const double s6 = s2 * s2 * s2;
                const double coef = 24.0 * eps * inv2 * (2.0 * s6 * s6 - s6);
                const double e = 4.0 * eps * (s6 * s6 - s6);
                return {std::fabs(coef) * std::sqrt(a.d2), std::fabs(e)};
            });
        const sfcnl_ref::PassConfig cfg(query_scale, sfcnl_ref::Isa::automatic, threads);
        const auto r = sfcnl_ref::reduce<double>(ps, box, store, k, cfg);
        std::memcpy(absf, r.outputs[0].data(), n * 8);
        std::memcpy(abse, r.outputs[1].data(), n * 8);
    });
}
