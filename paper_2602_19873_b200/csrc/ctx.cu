// C-ABI entry points (include/sfcnl_cu.h): context lifetime, uploads/downloads,
// error mapping, stage timing. Each entry point forwards to a kernel driver.
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ctx.hpp"

using namespace sfcnl_cu;

namespace sfcnl_cu {

namespace {
thread_local sfcnl_cu_ctx* g_cur = nullptr;  // context of the call in progress
thread_local std::string g_create_err;
}  // namespace

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    if (g_cur) {
        g_cur->err = buf;
        g_cur->err_off = 0;
    } else {
        g_create_err = buf;
    }
    return SFCNL_CUDA_ERROR;
}

int set_error(sfcnl_cu_ctx* c, int code, const std::string& msg, uint64_t off) {
    c->err = msg;
    c->err_off = off;
    return code;
}

int check_dev_error(sfcnl_cu_ctx* c, const char* const* messages) {
    DevError e;
    SFCNL_CUDA_TRY(cudaMemcpyAsync(&e, c->derr.p, sizeof e, cudaMemcpyDeviceToHost, c->stream));
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (e.key == ~0ull) return 0;
    const int code = int(e.key & 0xff);
    const int status = code >> 4, msg = code & 15;
    std::string text = messages[msg];
    if (status == SFCNL_DECODE_ERROR) text += " (byte offset " + std::to_string(e.offset) + ")";
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    return set_error(c, status, text, e.offset);
}

void stage_begin(sfcnl_cu_ctx* c, Stage s) {
    if (c->timing) {
        cudaEventRecord(c->ev[2 * s], c->stream);
        c->stage_pending[s] = true;
    }
}

void stage_end(sfcnl_cu_ctx* c, Stage s) {
    if (c->timing) cudaEventRecord(c->ev[2 * s + 1], c->stream);
}

}  // namespace sfcnl_cu

namespace {

struct CallScope {
    explicit CallScope(sfcnl_cu_ctx* c) {
        g_cur = c;
        if (c) cudaSetDevice(c->device);
    }
    ~CallScope() { g_cur = nullptr; }
};

Box make_box(const sfcnl_box* b) {
    Box r{};
    for (int d = 0; d < 3; ++d) {
        r.lo[d] = b->lo[d];
        r.hi[d] = b->hi[d];
        r.len[d] = b->hi[d] - b->lo[d];
        r.per[d] = b->periodic[d] != 0;
    }
    return r;
}

int check_box(sfcnl_cu_ctx* c, const sfcnl_box* b) {
    if (!b) return set_error(c, SFCNL_INPUT_ERROR, "null box");
    for (int d = 0; d < 3; ++d)
        if (!(b->hi[d] > b->lo[d]))
            return set_error(c, SFCNL_INPUT_ERROR, "SimulationBox: hi must exceed lo on every axis");
    return 0;
}

int upload(sfcnl_cu_ctx* c, DBuf& dst, const void* src, size_t bytes) {
    SFCNL_CUDA_TRY(dst.reserve(bytes));
    if (bytes) SFCNL_CUDA_TRY(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return 0;
}

int set_slot(sfcnl_cu_ctx* c, Slot& s, uint64_t n, const double* x, const double* y, const double* z,
             const double* h, const sfcnl_box* box) {
    if (int rc = check_box(c, box)) return rc;
    if (n && (!x || !y || !z || !h)) return set_error(c, SFCNL_INPUT_ERROR, "null particle array");
    s.valid = false;
    s.n = n;
    s.box = make_box(box);
    s.fields.clear();
    if (int rc = upload(c, s.x, x, n * 8)) return rc;
    if (int rc = upload(c, s.y, y, n * 8)) return rc;
    if (int rc = upload(c, s.z, z, n * 8)) return rc;
    if (int rc = upload(c, s.h, h, n * 8)) return rc;
    s.valid = true;
    return 0;
}

int set_slot_field(sfcnl_cu_ctx* c, Slot& s, const char* name, const double* v) {
    if (!s.valid) return set_error(c, SFCNL_INPUT_ERROR, "set_field: no particles set");
    if (!name) return set_error(c, SFCNL_INPUT_ERROR, "set_field: null name");
    Field* f = s.find(name);
    if (!f) {
        s.fields.emplace_back();
        f = &s.fields.back();
        f->name = name;
    }
    return upload(c, f->data, v, s.n * 8);
}

int download(sfcnl_cu_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes && dst) SFCNL_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

int finish(sfcnl_cu_ctx* c) {
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return 0;
}

}  // namespace

extern "C" {

int sfcnl_cu_ctx_create(int device, sfcnl_cu_ctx** out) {
    CallScope scope(nullptr);
    if (!out) return SFCNL_INPUT_ERROR;
    *out = nullptr;
    int ndev = 0;
    SFCNL_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) {
        g_create_err = "sfcnl_cu_ctx_create: no such CUDA device";
        return SFCNL_CUDA_ERROR;
    }
    SFCNL_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    SFCNL_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        g_create_err = "sfcnl_cu_ctx_create: this build targets sm_100a (B200); found sm_" +
                       std::to_string(prop.major) + std::to_string(prop.minor);
        return SFCNL_CUDA_ERROR;
    }
    auto* c = new (std::nothrow) sfcnl_cu_ctx();
    if (!c) return SFCNL_CUDA_ERROR;
    g_cur = c;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    SFCNL_CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) SFCNL_CUDA_TRY(cudaEventCreate(&e));
    SFCNL_CUDA_TRY(c->derr.reserve(sizeof(DevError)));
    SFCNL_CUDA_TRY(cudaMemsetAsync(c->derr.p, 0xff, sizeof(DevError), c->stream));
    uint16_t table[48 * 8];
    hilbert_table(table);
    SFCNL_CUDA_TRY(c->hilbert_table.reserve(sizeof table));
    SFCNL_CUDA_TRY(cudaMemcpyAsync(c->hilbert_table.p, table, sizeof table, cudaMemcpyHostToDevice, c->stream));
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *out = c;
    return SFCNL_OK;
}

void sfcnl_cu_ctx_destroy(sfcnl_cu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* sfcnl_cu_last_error(sfcnl_cu_ctx* c, uint64_t* byte_offset) {
    if (!c) {
        if (byte_offset) *byte_offset = 0;
        return g_create_err.c_str();
    }
    if (byte_offset) *byte_offset = c->err_off;
    return c->err.c_str();
}

void* sfcnl_cu_stream(sfcnl_cu_ctx* c) { return c ? (void*)c->stream : nullptr; }

int sfcnl_cu_synchronize(sfcnl_cu_ctx* c) {
    CallScope scope(c);
    return finish(c);
}

uint64_t sfcnl_cu_launch_count(sfcnl_cu_ctx* c) { return c ? c->launches : 0; }

int sfcnl_cu_set_timing(sfcnl_cu_ctx* c, int enabled) {
    c->timing = enabled != 0;
    for (auto& p : c->stage_pending) p = false;
    return 0;
}

int sfcnl_cu_stage_times(sfcnl_cu_ctx* c, double* ms, int cap) {
    CallScope scope(c);
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    int k = 0;
    for (; k < kNumStages && k < cap; ++k) {
        float v = 0.f;
        if (c->stage_pending[k]) cudaEventElapsedTime(&v, c->ev[2 * k], c->ev[2 * k + 1]);
        ms[k] = v;
    }
    return k;
}

int sfcnl_cu_set_particles(sfcnl_cu_ctx* c, uint64_t n, const double* x, const double* y,
                           const double* z, const double* h, const sfcnl_box* box) {
    CallScope scope(c);
    c->has_order = false;
    if (int rc = set_slot(c, c->orig, n, x, y, z, h, box)) return rc;
    return finish(c);
}

int sfcnl_cu_set_field(sfcnl_cu_ctx* c, const char* name, const double* v) {
    CallScope scope(c);
    if (int rc = set_slot_field(c, c->orig, name, v)) return rc;
    return finish(c);
}

int sfcnl_cu_set_sorted_particles(sfcnl_cu_ctx* c, uint64_t n, const double* x, const double* y,
                                  const double* z, const double* h, const sfcnl_box* box) {
    CallScope scope(c);
    if (int rc = set_slot(c, c->sorted, n, x, y, z, h, box)) return rc;
    return finish(c);
}

int sfcnl_cu_set_sorted_field(sfcnl_cu_ctx* c, const char* name, const double* v) {
    CallScope scope(c);
    if (int rc = set_slot_field(c, c->sorted, name, v)) return rc;
    return finish(c);
}

int sfcnl_cu_sort_by_sfc(sfcnl_cu_ctx* c, int bits) {
    CallScope scope(c);
    if (int rc = run_sort_by_sfc(c, bits)) return rc;
    return finish(c);
}

int sfcnl_cu_get_order(sfcnl_cu_ctx* c, uint64_t* keys, uint32_t* perm) {
    CallScope scope(c);
    if (!c->has_order) return set_error(c, SFCNL_INPUT_ERROR, "get_order: no SFC order");
    if (int rc = download(c, keys, c->keys.p, c->order_n * 8)) return rc;
    if (int rc = download(c, perm, c->perm.p, c->order_n * 4)) return rc;
    return finish(c);
}

int sfcnl_cu_set_order(sfcnl_cu_ctx* c, uint64_t n, const uint64_t* keys, const uint32_t* perm, int bits) {
    CallScope scope(c);
    if (bits < 1 || bits > 21) return set_error(c, SFCNL_INPUT_ERROR, "bits per dimension must be in [1, 21]");
    if (int rc = upload(c, c->keys, keys, n * 8)) return rc;
    if (perm) {
        if (int rc = upload(c, c->perm, perm, n * 4)) return rc;
    } else {
        SFCNL_CUDA_TRY(c->perm.reserve(std::max<uint64_t>(n, 1) * 4));
    }
    c->order_n = n;
    c->bits = bits;
    c->has_order = true;
    c->has_tree = false;
    return finish(c);
}

int sfcnl_cu_apply_order(sfcnl_cu_ctx* c) {
    CallScope scope(c);
    if (int rc = run_apply_order(c)) return rc;
    return finish(c);
}

int sfcnl_cu_get_sorted(sfcnl_cu_ctx* c, const char* name, double* out) {
    CallScope scope(c);
    Slot& s = c->sorted;
    if (!s.valid) return set_error(c, SFCNL_INPUT_ERROR, "get_sorted: no sorted particles");
    const std::string nm = name ? name : "";
    const DBuf* b = nm == "x" ? &s.x : nm == "y" ? &s.y : nm == "z" ? &s.z : nm == "h" ? &s.h : nullptr;
    if (!b) {
        Field* f = s.find(nm);
        if (!f) return set_error(c, SFCNL_INPUT_ERROR, "ParticleSet: no such field: " + nm);
        b = &f->data;
    }
    if (int rc = download(c, out, b->p, s.n * 8)) return rc;
    return finish(c);
}

int sfcnl_cu_build_octree(sfcnl_cu_ctx* c, uint32_t bucket, uint64_t* num_nodes) {
    CallScope scope(c);
    if (int rc = run_build_octree(c, bucket)) return rc;
    if (num_nodes) *num_nodes = c->num_nodes;
    return finish(c);
}

int sfcnl_cu_get_octree(sfcnl_cu_ctx* c, sfcnl_node* nodes) {
    CallScope scope(c);
    if (!c->has_tree) return set_error(c, SFCNL_INPUT_ERROR, "get_octree: no octree");
    if (int rc = download(c, nodes, c->nodes.p, c->num_nodes * sizeof(Node))) return rc;
    return finish(c);
}

int sfcnl_cu_set_octree(sfcnl_cu_ctx* c, uint64_t num_nodes, const sfcnl_node* nodes, int bits, uint64_t n) {
    CallScope scope(c);
    static_assert(sizeof(sfcnl_node) == sizeof(Node), "node layout");
    if (num_nodes == 0 || !nodes) return set_error(c, SFCNL_INPUT_ERROR, "set_octree: empty tree");
    for (uint64_t k = 0; k < num_nodes; ++k) {
        const int32_t fc = nodes[k].first_child;
        if (fc >= 0 && (uint64_t(fc) <= k || uint64_t(fc) + 8 > num_nodes))
            return set_error(c, SFCNL_BUILD_ERROR, "set_octree: malformed node array");
    }
    if (int rc = upload(c, c->nodes, nodes, num_nodes * sizeof(Node))) return rc;
    std::vector<uint8_t> depth(num_nodes);
    for (uint64_t k = 0; k < num_nodes; ++k) depth[k] = nodes[k].depth;
    c->num_nodes = num_nodes;
    c->tree_bits = bits;
    c->tree_n = n;
    c->has_tree = true;
    if (int rc = run_tree_levels_from_nodes(c, depth)) return rc;
    return finish(c);
}

int sfcnl_cu_node_geometry(sfcnl_cu_ctx* c, double* lo, double* hi, double* radius) {
    CallScope scope(c);
    if (int rc = run_node_geometry(c)) return rc;
    std::vector<Geo> g(c->num_nodes);
    if (int rc = download(c, g.data(), c->node_geo.p, c->num_nodes * sizeof(Geo))) return rc;
    if (int rc = finish(c)) return rc;
    for (uint64_t k = 0; k < c->num_nodes; ++k) {
        for (int d = 0; d < 3; ++d) {
            if (lo) lo[3 * k + d] = g[k].lo[d];
            if (hi) hi[3 * k + d] = g[k].hi[d];
        }
        if (radius) radius[k] = g[k].maxh;
    }
    return 0;
}

int sfcnl_cu_build_store(sfcnl_cu_ctx* c, const sfcnl_build_params* p, uint64_t* num_sc,
                         uint64_t* blob_bytes) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null build params");
    if (int rc = run_build_store(c, *p)) return rc;
    if (num_sc) *num_sc = c->num_sc;
    if (blob_bytes) *blob_bytes = c->blob_bytes;
    return finish(c);
}

int sfcnl_cu_get_store(sfcnl_cu_ctx* c, uint32_t* counts, uint64_t* offsets, uint8_t* blob) {
    CallScope scope(c);
    if (!c->has_store) return set_error(c, SFCNL_INPUT_ERROR, "get_store: no store");
    if (int rc = download(c, counts, c->counts.p, c->num_sc * 4)) return rc;
    if (int rc = download(c, offsets, c->offsets.p, (c->num_sc + 1) * 8)) return rc;
    if (int rc = download(c, blob, c->blob.p, c->blob_bytes)) return rc;
    return finish(c);
}

int sfcnl_cu_set_store(sfcnl_cu_ctx* c, const sfcnl_build_params* p, uint64_t n, uint64_t num_sc,
                       const uint32_t* counts, const uint64_t* offsets, const uint8_t* blob,
                       uint64_t blob_bytes) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null build params");
    if (p->ci == 0 || p->cj == 0 || 64 % p->ci || 64 % p->cj || p->ci % p->cj || (p->w != 32 && p->w != 64))
        return set_error(c, SFCNL_INPUT_ERROR, "ClusterParams: invalid cluster parameters");
    if (num_sc != (n + 63) / 64) return set_error(c, SFCNL_INPUT_ERROR, "set_store: super-cluster count mismatch");
    for (uint64_t s = 0; s < num_sc; ++s)
        if (offsets[s + 1] < offsets[s] || offsets[s + 1] > blob_bytes)
            return set_error(c, SFCNL_DECODE_ERROR, "set_store: offsets out of range", offsets[s]);
    if (int rc = upload(c, c->counts, counts, num_sc * 4)) return rc;
    if (int rc = upload(c, c->offsets, offsets, (num_sc + 1) * 8)) return rc;
    if (int rc = upload(c, c->blob, blob, blob_bytes)) return rc;
    c->sp = *p;
    c->store_n = n;
    c->num_sc = num_sc;
    c->blob_bytes = blob_bytes;
    c->has_store = true;
    c->btab_valid = false;  // rebuilt on demand by the pass
    return finish(c);
}

int sfcnl_cu_reduce(sfcnl_cu_ctx* c, const sfcnl_pass_params* p, double* const* outs, uint32_t* count) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null pass params");
    if (int rc = run_reduce(c, *p)) return rc;
    const int no = p->kernel >= 2 ? 4 : 1;
    const uint64_t n = c->sorted.n;
    if (outs)
        for (int o = 0; o < no; ++o)
            if (int rc = download(c, outs[o], c->outs[o].p, n * 8)) return rc;
    if (int rc = download(c, count, c->ncount.p, n * 4)) return rc;
    return finish(c);
}

}  // extern "C"
