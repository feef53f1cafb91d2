// Context object behind the C-ABI (include/sfcnl_cu.h): owns the stream, the
// device copies of the particle slots and every derived structure.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sfcnl_cu {

// Device bytes held by every DBuf of the process (sfcnl_cu_memory_bytes).
uint64_t& dbuf_total_bytes();

// Grow-only device allocation: the hot path reuses buffers across steps.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, bytes = o.bytes;
            o.p = nullptr, o.bytes = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p), dbuf_total_bytes() -= bytes;
        p = nullptr;
        bytes = 0;
    }
    cudaError_t reserve(size_t b) {
        if (b <= bytes && p) return cudaSuccess;
        release();
        const size_t want = b ? b : 16;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) bytes = want, dbuf_total_bytes() += want;
        else p = nullptr;
        return e;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct Field {
    std::string name;
    DBuf data;
};

struct Slot {
    uint64_t n = 0;
    bool valid = false;
    Box box{};
    DBuf x, y, z, h;
    std::vector<Field> fields;
    Field* find(const std::string& name) {
        for (auto& f : fields)
            if (f.name == name) return &f;
        return nullptr;
    }
};

enum Stage { kKeygen, kSort, kPermute, kOctree, kNodeGeo, kClusterGeo, kBuild, kEncode, kPass, kNumStages };

}  // namespace sfcnl_cu

struct sfcnl_cu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t err_off = 0;
    uint64_t launches = 0;
    int num_sms = 148;

    sfcnl_cu::Slot orig, sorted;
    std::vector<sfcnl_cu::Field> field_pool;  // allocations of fields dropped by set_particles, reused by name

    // (1) order
    bool has_order = false;
    int bits = 21;
    uint64_t order_n = 0;
    sfcnl_cu::DBuf keys, perm, keys_alt, perm_alt;
    sfcnl_cu::DBuf records;  // apply_order: packed particle records (sfc_sort.cu)
    sfcnl_cu::DBuf hist, digit_base, status, tile_counter;
    sfcnl_cu::DBuf hilbert_table;

    // (3) octree
    bool has_tree = false;
    int tree_bits = 21;
    uint64_t tree_n = 0;
    uint64_t num_nodes = 0;
    sfcnl_cu::DBuf nodes;      // sfcnl_cu::Node[num_nodes]
    sfcnl_cu::DBuf level_nodes;  // node indices grouped by depth (deepest processed first)
    std::vector<uint64_t> level_off;  // host: level d occupies [level_off[d], level_off[d+1])
    sfcnl_cu::DBuf node_geo;   // Geo[num_nodes]
    sfcnl_cu::DBuf node_geo32; // node boxes in fp32 for the build traversal's pre-test
    bool node_geo_external = false;  // node_geo supplied by the caller (domain decomposition)
    sfcnl_cu::DBuf tree_scratch;
    // level-synchronous construction scratch, one entry per depth
    struct Level {
        sfcnl_cu::DBuf kf, pb, pe, flag, ipos, ikeys, irank;
        sfcnl_cu::DBuf g;  // distributed build: global particle ranges [pb | pe] (all-reduced local bounds)
        uint64_t count = 0, internal = 0;
    };
    std::vector<Level> levels;
    sfcnl_cu::DBuf level_tab;  // device table of per-level ikeys pointers + counts

    // (2) clusters
    sfcnl_cu::DBuf igeo, jgeo;

    // (4) store
    bool has_store = false;
    uint64_t store_gen = 0;                   // bumped whenever the store changes
    sfcnl_cu::DBuf dec_idx, dec_base;         // the store's decoded index lists (pass.cu), for store_gen
    uint64_t dec_gen = ~0ull;
    sfcnl_build_params sp{};
    bool clgeo_whole = false;  // igeo/jgeo hold every cluster of the current sorted set (device_array)
    uint64_t store_n = 0, num_sc = 0, blob_bytes = 0;
    sfcnl_cu::DBuf counts, offsets, blob;
    uint64_t sc_base = 0;  // first (global) super-cluster of the current store
    sfcnl_cu::DBuf jflags;  // halo: u8 per global j-cluster, set by run_halo_mark
    bool jflags_valid = false;
    uint64_t jflags_sc0 = 0, jflags_sc1 = 0, jflags_len = 0;
    sfcnl_cu::DBuf leaf_cache, leaf_count;  // accepted leaves per SC from halo_mark (reused by the range build)
    bool leaf_cache_valid = false;
    sfcnl_cu::DBuf sc_size, sc_scratch_off, scratch, build_ctl, overflow_list, fallback_ws;

    // (5) pass
    sfcnl_cu::DBuf outs[4], ncount, jstage;
    sfcnl_cu::DBuf work_ctr;  // dynamic work counter of the warp-per-SC kernels
    sfcnl_cu::DBuf frame, frame_x, frame_xcl;  // cluster-frame fp32 positions (+ payload), max |offset| per axis (frame.cu)

    // full Verlet list baseline (pass_full.cuh): CSR offsets u64[n+1], neighbors u32
    bool has_full = false;
    uint64_t full_n = 0, full_pairs = 0;
    double full_scale = 0;
    int full_mode = 0;
    sfcnl_cu::DBuf full_cnt, full_off, full_nbr;
    // symmetric pass (pass_sym.cuh): entry base, j-side accumulators/counts, entry
    // j-cluster/SC, transposed entry lists per j-cluster
    sfcnl_cu::DBuf sym[9];
    sfcnl_cu::DBuf sym_aux, sym_spec;
    sfcnl_cu::DBuf symc[4];  // domain decomposition: remote + local entry accumulators (sym_range_final)
    uint64_t sym_e_local = 0;
    int sym_e_kernel = -1;  // + fp64 j-side sums of the deferred special slots  // symmetric mixed density: per-particle error-bound weights (+ flag counter)
    uint64_t last_redo = 0;  // particles / SCs handed to fp64 by the last mixed pass's error bound  // [8]: deferred special-slot queues of the symmetric fast pass

    // O(N/P) domain decomposition (dd.cu): local cluster -> global id (encoder) and
    // global -> local cluster (pass decoders), caller-owned device arrays; null = off
    const uint32_t* dd_lc2g = nullptr;
    const uint32_t* dd_g2l = nullptr;
    sfcnl_cu::DBuf dd_tab;  // device pointer tables / small scratch of the dd kernels

    // errors
    sfcnl_cu::DBuf derr;  // DevError
    sfcnl_cu::DBuf ptrs;  // small pointer tables
    sfcnl_cu::DBuf scan_tmp;
    sfcnl_cu::DBuf small_host_dev;  // tiny device scratch for readbacks
    void* hmap = nullptr;            // mapped pinned host page for small readbacks (no copy engine)
    void* dmap = nullptr;            // its device alias

    // timing
    bool timing = false;
    cudaEvent_t ev[2 * sfcnl_cu::kNumStages] = {};
    float stage_ms[sfcnl_cu::kNumStages] = {};
    bool stage_pending[sfcnl_cu::kNumStages] = {};
};

namespace sfcnl_cu {

int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
int set_error(sfcnl_cu_ctx* c, int code, const std::string& msg, uint64_t off = 0);
int check_dev_error(sfcnl_cu_ctx* c, const char* const* messages);
// Small device -> host readback (<= 64 KB) written by a kernel into a mapped pinned page:
// it does not queue behind bulk transfers on the copy engines (StreamedPipeline). Syncs
// the context's stream.
int readback(sfcnl_cu_ctx* c, void* dst, const void* src, size_t bytes);

void stage_begin(sfcnl_cu_ctx* c, Stage s);
void stage_end(sfcnl_cu_ctx* c, Stage s);

// Kernel drivers (each in its own .cu).
int run_sort_by_sfc(sfcnl_cu_ctx* c, int bits);
int run_apply_order(sfcnl_cu_ctx* c, int64_t into = -1);  // into >= 0: gather into sorted[into..]
// Distributed octree (domain decomposition): every rank holds a disjoint part of the
// global key multiset in c->keys (sorted); a node's global particle bound is the sum over
// ranks of the local lower bounds, so each level's child bounds are all-reduced (SUM) by
// the caller's collective and the result is the single-domain tree on every rank.
struct DistTree {
    uint64_t n_global;
    sfcnl_allreduce_u32 fn;  // in-place SUM over ranks of `count` u32 on the device
    void* user;
};
int run_build_octree(sfcnl_cu_ctx* c, uint32_t bucket, const DistTree* dt = nullptr);
int run_tree_levels_from_nodes(sfcnl_cu_ctx* c, const std::vector<uint8_t>& depth);
int run_node_geometry(sfcnl_cu_ctx* c, uint64_t p0 = 0, uint64_t p1 = ~0ull);  // leaves clip to [p0, p1)
// clusters overlapping particles [p0, p1), plus j-clusters flagged in jflags (if non-null)
int run_cluster_geometry(sfcnl_cu_ctx* c, uint32_t ci, uint32_t cj, uint64_t p0 = 0, uint64_t p1 = ~0ull,
                         const uint8_t* jflags = nullptr);
int run_build_store(sfcnl_cu_ctx* c, const sfcnl_build_params& p, uint64_t sc0, uint64_t sc1, double max_h);
int run_reduce(sfcnl_cu_ctx* c, const sfcnl_pass_params& p);
int run_build_full_list(sfcnl_cu_ctx* c, double build_scale);
int run_reduce_full(sfcnl_cu_ctx* c, const sfcnl_pass_params& p);
int run_cluster_slots(sfcnl_cu_ctx* c, uint64_t* slots);
int run_sym_range_entries(sfcnl_cu_ctx* c, const sfcnl_pass_params& p, uint64_t* num_e);
int run_sym_range_final(sfcnl_cu_ctx* c, const sfcnl_pass_params& p, uint64_t nr, const double* rjacc,
                        const uint32_t* rjcnt, const uint32_t* rejcl, const uint32_t* resc);
// cluster-frame staging copy of the sorted positions (frame.cu); m = payload or null
// clusters overlapping particles [p_lo, p_hi) plus those flagged in jflags (if non-null)
int run_frame(sfcnl_cu_ctx* c, uint32_t cj, const double* m, uint64_t p_lo = 0, uint64_t p_hi = ~0ull,
              const uint8_t* jflags = nullptr);
int run_halo_mark(sfcnl_cu_ctx* c, const sfcnl_build_params& p, uint64_t sc0, uint64_t sc1);

// Host helpers shared with the C++ drop-in.
void hilbert_table(uint16_t* table);  // 48 states x 8 octants: out | next << 3
int host_set_error(int code, const std::string& msg, uint64_t off = 0);

// Caller-supplied node geometry and halo flags describe one tree + particle set.
inline void drop_external(sfcnl_cu_ctx* c) {
    c->node_geo_external = false;
    c->jflags_valid = false;
    c->leaf_cache_valid = false;
}

// Particles covered by the current store's super-cluster range (outputs of a pass).
inline uint64_t pass_out_count(const sfcnl_cu_ctx* c) {
    const uint64_t lo = c->sc_base * 64;
    const uint64_t hi = std::min<uint64_t>(c->sorted.n, (c->sc_base + c->num_sc) * 64);
    return hi > lo ? hi - lo : 0;
}

template <class K, class... A>
inline void launch(sfcnl_cu_ctx* c, K kernel, dim3 grid, dim3 block, size_t smem, A... args) {
    kernel<<<grid, block, smem, c->stream>>>(args...);
    ++c->launches;
}

}  // namespace sfcnl_cu
