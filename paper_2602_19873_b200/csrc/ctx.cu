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

constexpr size_t kMapBytes = 64 * 1024;

__global__ void k_readback(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, size_t bytes) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < bytes; k += size_t(gridDim.x) * blockDim.x)
        dst[k] = src[k];
}

int readback(sfcnl_cu_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return 0;
    if (!c->hmap || bytes > kMapBytes) {  // fallback: the copy engine
        SFCNL_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        return 0;
    }
    k_readback<<<unsigned(std::min<size_t>((bytes + 255) / 256, 64)), 256, 0, c->stream>>>(
        static_cast<const unsigned char*>(src), static_cast<unsigned char*>(c->dmap), bytes);
    SFCNL_CUDA_TRY(cudaGetLastError());
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::memcpy(dst, c->hmap, bytes);
    return 0;
}

int check_dev_error(sfcnl_cu_ctx* c, const char* const* messages) {
    DevError e;
    if (int rc = readback(c, &e, c->derr.p, sizeof e)) return rc;
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

// Row-major [n, ncols] records -> ncols SoA columns (one pass).
__global__ void k_unpack_records(uint64_t n, int ncols, const double* __restrict__ rec, double* const* __restrict__ dst) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x)
        for (int a = 0; a < ncols; ++a) dst[a][k] = rec[k * ncols + a];
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
    // cudaMemcpyDefault: the source may be host (pageable/pinned) or device memory (UVA)
    if (bytes) SFCNL_CUDA_TRY(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyDefault, c->stream));
    return 0;
}

int set_slot(sfcnl_cu_ctx* c, Slot& s, uint64_t n, const double* x, const double* y, const double* z,
             const double* h, const sfcnl_box* box) {
    if (int rc = check_box(c, box)) return rc;
    if (n && (!x || !y || !z || !h)) return set_error(c, SFCNL_INPUT_ERROR, "null particle array");
    // particle indices are 32-bit throughout the reference (SfcOrder::perm, OctreeNode
    // particle ranges, j-cluster indices): 2^32 - 1 particles at most
    if (n > 0xffffffffull) return set_error(c, SFCNL_INPUT_ERROR, "ParticleSet: more than 2^32 - 1 particles");
    s.valid = false;
    s.n = n;
    s.box = make_box(box);
    // keep the field allocations for the next set_field of the same name (no cudaFree/cudaMalloc per step)
    for (auto& f : s.fields) c->field_pool.push_back(std::move(f));
    s.fields.clear();
    drop_external(c);
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
        for (auto it = c->field_pool.begin(); it != c->field_pool.end(); ++it)
            if (it->name == f->name) {
                f->data = std::move(it->data);
                c->field_pool.erase(it);
                break;
            }
    }
    return upload(c, f->data, v, s.n * 8);
}

int download(sfcnl_cu_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes && dst) SFCNL_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
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
    if (cudaHostAlloc(&c->hmap, kMapBytes, cudaHostAllocMapped) == cudaSuccess) {
        if (cudaHostGetDevicePointer(&c->dmap, c->hmap, 0) != cudaSuccess) {
            cudaFreeHost(c->hmap);
            c->hmap = c->dmap = nullptr;
        }
    } else {
        cudaGetLastError();
        c->hmap = nullptr;
    }
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
    if (c->hmap) cudaFreeHost(c->hmap);
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

int sfcnl_cu_set_particle_records(sfcnl_cu_ctx* c, uint64_t n, const double* rec, int ncols,
                                  const char* const* fields, const sfcnl_box* box) {
    CallScope scope(c);
    if (ncols < 4) return set_error(c, SFCNL_INPUT_ERROR, "set_particle_records: need x, y, z, h columns");
    if (n && !rec) return set_error(c, SFCNL_INPUT_ERROR, "null particle array");
    if (int rc = check_box(c, box)) return rc;
    Slot& s = c->orig;
    c->has_order = false;
    s.valid = false;
    s.n = n;
    s.box = make_box(box);
    drop_external(c);
    SFCNL_CUDA_TRY(s.x.reserve(n * 8));
    SFCNL_CUDA_TRY(s.y.reserve(n * 8));
    SFCNL_CUDA_TRY(s.z.reserve(n * 8));
    SFCNL_CUDA_TRY(s.h.reserve(n * 8));
    std::vector<Field> nf(ncols - 4);
    for (int k = 0; k < ncols - 4; ++k) {
        if (!fields || !fields[k]) return set_error(c, SFCNL_INPUT_ERROR, "set_particle_records: null field name");
        nf[k].name = fields[k];
        if (Field* old = s.find(fields[k])) nf[k].data = std::move(old->data);
        SFCNL_CUDA_TRY(nf[k].data.reserve(n * 8));
    }
    s.fields = std::move(nf);
    std::vector<void*> host{s.x.p, s.y.p, s.z.p, s.h.p};
    for (auto& f : s.fields) host.push_back(f.data.p);
    SFCNL_CUDA_TRY(c->ptrs.reserve(ncols * sizeof(void*)));
    SFCNL_CUDA_TRY(cudaMemcpyAsync(c->ptrs.p, host.data(), ncols * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    if (n) {
        const int grid = int(std::min<uint64_t>((n + 255) / 256, uint64_t(c->num_sms) * 16));
        launch(c, k_unpack_records, dim3(grid), dim3(256), 0, n, ncols, rec, (double* const*)c->ptrs.as<void*>());
        SFCNL_CUDA_TRY(cudaGetLastError());
    }
    s.valid = true;
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
    drop_external(c);
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
    if (int rc = run_build_store(c, *p, 0, ~0ull, 0.0)) return rc;
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
    c->clgeo_whole = false;
    c->store_n = n;
    c->num_sc = num_sc;
    c->blob_bytes = blob_bytes;
    c->has_store = true;
    ++c->store_gen;
    c->sc_base = 0;
    return finish(c);
}

int sfcnl_cu_get_device_view(sfcnl_cu_ctx* c, sfcnl_cu_device_view* v) {
    CallScope scope(c);
    if (!v) return set_error(c, SFCNL_INPUT_ERROR, "null device view");
    if (!c->sorted.valid) return set_error(c, SFCNL_INPUT_ERROR, "device view: no particles");
    if (!c->has_store) return set_error(c, SFCNL_INPUT_ERROR, "device view: no neighbor store");
    if (c->store_n != c->sorted.n) return set_error(c, SFCNL_INPUT_ERROR, "reduce: store/particle-set size mismatch");
    if (c->sc_base != 0 || c->num_sc != (c->sorted.n + 63) / 64)
        return set_error(c, SFCNL_INPUT_ERROR, "device view: the store covers a super-cluster range");
    *v = sfcnl_cu_device_view{};
    v->n = c->sorted.n;
    v->num_sc = c->num_sc;
    v->ci = c->sp.ci, v->cj = c->sp.cj;
    v->w = c->sp.w, v->mode = c->sp.mode, v->compress = c->sp.compress;
    for (int d = 0; d < 3; ++d) v->box_len[d] = c->sorted.box.per[d] ? c->sorted.box.len[d] : 0.0;
    v->x = c->sorted.x.as<const double>(), v->y = c->sorted.y.as<const double>();
    v->z = c->sorted.z.as<const double>(), v->h = c->sorted.h.as<const double>();
    v->counts = c->counts.as<const uint32_t>(), v->offsets = c->offsets.as<const uint64_t>();
    v->blob = c->blob.as<const uint8_t>(), v->blob_bytes = c->blob_bytes;
    v->stream = (void*)c->stream;
    return finish(c);
}

int sfcnl_cu_sorted_field_ptr(sfcnl_cu_ctx* c, const char* name, const double** out) {
    CallScope scope(c);
    auto* f = c->sorted.find(name);
    if (!f) return set_error(c, SFCNL_INPUT_ERROR, std::string("ParticleSet: no such field: ") + name);
    *out = f->data.as<const double>();
    return finish(c);
}

int sfcnl_cu_reduce(sfcnl_cu_ctx* c, const sfcnl_pass_params* p, double* const* outs, uint32_t* count) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null pass params");
    if (int rc = run_reduce(c, *p)) return rc;
    const int no = p->kernel >= 2 ? 4 : 1;
    const uint64_t n = pass_out_count(c);
    if (outs)
        for (int o = 0; o < no; ++o)
            if (int rc = download(c, outs[o], c->outs[o].p, n * 8)) return rc;
    if (int rc = download(c, count, c->ncount.p, n * 4)) return rc;
    return finish(c);
}

int sfcnl_cu_build_full_list(sfcnl_cu_ctx* c, double build_scale, uint64_t* num_pairs) {
    CallScope scope(c);
    if (int rc = run_build_full_list(c, build_scale)) return rc;
    if (num_pairs) *num_pairs = c->full_pairs;
    return finish(c);
}

int sfcnl_cu_get_full_list(sfcnl_cu_ctx* c, uint64_t* offsets, uint32_t* neighbors) {
    CallScope scope(c);
    if (!c->has_full) return set_error(c, SFCNL_INPUT_ERROR, "get_full_list: no full list");
    if (int rc = download(c, offsets, c->full_off.p, (c->full_n + 1) * 8)) return rc;
    if (int rc = download(c, neighbors, c->full_nbr.p, c->full_pairs * 4)) return rc;
    return finish(c);
}

int sfcnl_cu_set_full_list(sfcnl_cu_ctx* c, uint64_t n, int mode, double build_scale, const uint64_t* offsets,
                           const uint32_t* neighbors, uint64_t num_pairs) {
    CallScope scope(c);
    if (mode != 0 && mode != 1) return set_error(c, SFCNL_INPUT_ERROR, "set_full_list: unknown list mode");
    if (!offsets) return set_error(c, SFCNL_INPUT_ERROR, "set_full_list: null offsets");
    if (offsets[0] != 0 || offsets[n] != num_pairs)
        return set_error(c, SFCNL_INPUT_ERROR, "set_full_list: offsets do not span the neighbor array");
    for (uint64_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return set_error(c, SFCNL_INPUT_ERROR, "set_full_list: offsets not monotone");
    for (uint64_t k = 0; k < num_pairs; ++k)
        if (neighbors[k] >= n) return set_error(c, SFCNL_INPUT_ERROR, "set_full_list: neighbor index out of range");
    c->has_full = false;
    if (int rc = upload(c, c->full_off, offsets, (n + 1) * 8)) return rc;
    if (int rc = upload(c, c->full_nbr, neighbors, num_pairs * 4)) return rc;
    c->full_n = n, c->full_pairs = num_pairs, c->full_scale = build_scale, c->full_mode = mode;
    c->has_full = true;
    return finish(c);
}

int sfcnl_cu_reduce_full(sfcnl_cu_ctx* c, const sfcnl_pass_params* p, double* const* outs, uint32_t* count) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null pass params");
    if (int rc = run_reduce_full(c, *p)) return rc;
    const int no = p->kernel >= 2 ? 4 : 1;
    const uint64_t n = c->sorted.n;
    if (outs)
        for (int o = 0; o < no; ++o)
            if (int rc = download(c, outs[o], c->outs[o].p, n * 8)) return rc;
    if (int rc = download(c, count, c->ncount.p, n * 4)) return rc;
    return finish(c);
}

int sfcnl_cu_cluster_slots(sfcnl_cu_ctx* c, uint64_t* slots) {
    CallScope scope(c);
    uint64_t v = 0;
    if (int rc = run_cluster_slots(c, &v)) return rc;
    if (slots) *slots = v;
    return finish(c);
}

int sfcnl_cu_sym_range_entries(sfcnl_cu_ctx* c, const sfcnl_pass_params* p, uint64_t* num_entries) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null pass params");
    uint64_t ne = 0;
    if (int rc = run_sym_range_entries(c, *p, &ne)) return rc;
    if (num_entries) *num_entries = ne;
    return finish(c);
}

int sfcnl_cu_sym_range_final(sfcnl_cu_ctx* c, const sfcnl_pass_params* p, uint64_t num_remote, const double* jacc,
                             const uint32_t* jcnt, const uint32_t* ejcl, const uint32_t* esc, double* const* outs,
                             uint32_t* count) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null pass params");
    if (int rc = run_sym_range_final(c, *p, num_remote, jacc, jcnt, ejcl, esc)) return rc;
    const int no = p->kernel >= 2 ? 4 : 1;
    const uint64_t n = pass_out_count(c);
    if (outs)
        for (int o = 0; o < no; ++o)
            if (int rc = download(c, outs[o], c->outs[o].p, n * 8)) return rc;
    if (int rc = download(c, count, c->ncount.p, n * 4)) return rc;
    return finish(c);
}

int sfcnl_cu_build_store_range(sfcnl_cu_ctx* c, const sfcnl_build_params* p, uint64_t sc_begin, uint64_t sc_end,
                               double max_h, uint64_t* num_sc, uint64_t* blob_bytes) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null build params");
    if (int rc = run_build_store(c, *p, sc_begin, sc_end, max_h)) return rc;
    if (num_sc) *num_sc = c->num_sc;
    if (blob_bytes) *blob_bytes = c->blob_bytes;
    return finish(c);
}

int sfcnl_cu_alloc_sorted(sfcnl_cu_ctx* c, uint64_t n, const sfcnl_box* box, const char* const* fields,
                          int nfields) {
    CallScope scope(c);
    if (int rc = check_box(c, box)) return rc;
    if (n > 0xffffffffull) return set_error(c, SFCNL_INPUT_ERROR, "ParticleSet: more than 2^32 - 1 particles");
    Slot& s = c->sorted;
    s.valid = false;
    s.n = n;
    s.box = make_box(box);
    c->has_store = false;
    ++c->store_gen;
    drop_external(c);
    for (DBuf* b : {&s.x, &s.y, &s.z, &s.h}) SFCNL_CUDA_TRY(b->reserve(std::max<uint64_t>(n, 1) * 8));
    // keep the allocations of fields that survive (steps re-allocate the same set)
    std::vector<Field> next(nfields > 0 ? nfields : 0);
    for (int k = 0; k < nfields; ++k) {
        if (!fields[k]) return set_error(c, SFCNL_INPUT_ERROR, "alloc_sorted: null field name");
        next[k].name = fields[k];
        if (Field* old = s.find(fields[k])) next[k].data = std::move(old->data);
        SFCNL_CUDA_TRY(next[k].data.reserve(std::max<uint64_t>(n, 1) * 8));
    }
    s.fields = std::move(next);
    s.valid = true;
    return finish(c);
}

static DBuf* sorted_array(sfcnl_cu_ctx* c, const char* name) {
    Slot& s = c->sorted;
    const std::string nm = name ? name : "";
    if (nm == "x") return &s.x;
    if (nm == "y") return &s.y;
    if (nm == "z") return &s.z;
    if (nm == "h") return &s.h;
    Field* f = s.find(nm);
    return f ? &f->data : nullptr;
}

int sfcnl_cu_write_sorted(sfcnl_cu_ctx* c, const char* name, uint64_t offset, uint64_t count, const double* src,
                          int src_on_device) {
    CallScope scope(c);
    DBuf* b = sorted_array(c, name);
    if (!c->sorted.valid || !b) return set_error(c, SFCNL_INPUT_ERROR, "write_sorted: no such sorted array");
    if (offset + count > c->sorted.n) return set_error(c, SFCNL_INPUT_ERROR, "write_sorted: range out of bounds");
    if (count)
        SFCNL_CUDA_TRY(cudaMemcpyAsync(b->as<double>() + offset, src, count * 8,
                                       src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    return finish(c);
}

int sfcnl_cu_read_sorted(sfcnl_cu_ctx* c, const char* name, uint64_t offset, uint64_t count, double* dst,
                         int dst_on_device) {
    CallScope scope(c);
    DBuf* b = sorted_array(c, name);
    if (!c->sorted.valid || !b) return set_error(c, SFCNL_INPUT_ERROR, "read_sorted: no such sorted array");
    if (offset + count > c->sorted.n) return set_error(c, SFCNL_INPUT_ERROR, "read_sorted: range out of bounds");
    if (count)
        SFCNL_CUDA_TRY(cudaMemcpyAsync(dst, b->as<double>() + offset, count * 8,
                                       dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    return finish(c);
}

int sfcnl_cu_read_order(sfcnl_cu_ctx* c, uint64_t offset, uint64_t count, uint64_t* keys, uint32_t* perm,
                        int dst_on_device) {
    CallScope scope(c);
    if (!c->has_order || offset + count > c->order_n) return set_error(c, SFCNL_INPUT_ERROR, "read_order: bad range");
    const cudaMemcpyKind k = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (count && keys) SFCNL_CUDA_TRY(cudaMemcpyAsync(keys, c->keys.as<uint64_t>() + offset, count * 8, k, c->stream));
    if (count && perm) SFCNL_CUDA_TRY(cudaMemcpyAsync(perm, c->perm.as<uint32_t>() + offset, count * 4, k, c->stream));
    return finish(c);
}

int sfcnl_cu_set_keys(sfcnl_cu_ctx* c, uint64_t n, const uint64_t* keys, int src_on_device, int bits) {
    CallScope scope(c);
    if (bits < 1 || bits > 21) return set_error(c, SFCNL_INPUT_ERROR, "bits per dimension must be in [1, 21]");
    SFCNL_CUDA_TRY(c->keys.reserve(std::max<uint64_t>(n, 1) * 8));
    SFCNL_CUDA_TRY(c->perm.reserve(std::max<uint64_t>(n, 1) * 4));
    if (n)
        SFCNL_CUDA_TRY(cudaMemcpyAsync(c->keys.p, keys, n * 8,
                                       src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    c->order_n = n;
    c->bits = bits;
    c->has_order = true;
    c->has_tree = false;
    drop_external(c);
    return finish(c);
}

int sfcnl_cu_apply_order_into(sfcnl_cu_ctx* c, uint64_t offset) {
    CallScope scope(c);
    if (offset > (uint64_t(1) << 62)) return set_error(c, SFCNL_INPUT_ERROR, "apply_order_into: bad offset");
    if (int rc = run_apply_order(c, int64_t(offset))) return rc;
    return finish(c);
}

int sfcnl_cu_node_geometry_range(sfcnl_cu_ctx* c, uint64_t p_begin, uint64_t p_end) {
    CallScope scope(c);
    if (int rc = run_node_geometry(c, p_begin, p_end)) return rc;
    c->node_geo_external = true;
    return finish(c);
}

int sfcnl_cu_halo_mark(sfcnl_cu_ctx* c, const sfcnl_build_params* p, uint64_t sc_begin, uint64_t sc_end,
                       uint64_t* num_jclusters) {
    CallScope scope(c);
    if (!p) return set_error(c, SFCNL_INPUT_ERROR, "null build params");
    if (int rc = run_halo_mark(c, *p, sc_begin, sc_end)) return rc;
    if (num_jclusters) *num_jclusters = (c->sorted.n + p->cj - 1) / p->cj;
    return finish(c);
}

int sfcnl_cu_device_array(sfcnl_cu_ctx* c, const char* name, void** ptr, uint64_t* bytes) {
    CallScope scope(c);
    if (!name || !ptr) return set_error(c, SFCNL_INPUT_ERROR, "device_array: null argument");
    const std::string nm = name;
    DBuf* b = nullptr;
    uint64_t len = 0;
    if (nm == "keys" && c->has_order) b = &c->keys, len = c->order_n * 8;
    else if (nm == "perm" && c->has_order) b = &c->perm, len = c->order_n * 4;
    else if (nm == "node_geo" && c->has_tree) b = &c->node_geo, len = c->num_nodes * sizeof(Geo);
    else if (nm == "nodes" && c->has_tree) b = &c->nodes, len = c->num_nodes * sizeof(Node);
    else if (nm == "halo_flags" && c->jflags_valid) b = &c->jflags, len = c->jflags_len;
    // per-cluster geometry of the last build (compute_cluster_geometry, neighbor_build.cpp:19-38):
    // Geo {lo[3], hi[3], maxh, pad} per cluster; j-clusters alias i-clusters when ci == cj
    else if (nm == "cluster_geo.i" && c->has_store && c->clgeo_whole && c->sorted.valid)
        b = &c->igeo, len = (c->sorted.n + c->sp.ci - 1) / c->sp.ci * sizeof(Geo);
    else if (nm == "cluster_geo.j" && c->has_store && c->clgeo_whole && c->sorted.valid)
        b = c->sp.cj == c->sp.ci ? &c->igeo : &c->jgeo, len = (c->sorted.n + c->sp.cj - 1) / c->sp.cj * sizeof(Geo);
    else if (nm.rfind("out", 0) == 0 && nm.size() == 4 && nm[3] >= '0' && nm[3] <= '3')
        b = &c->outs[nm[3] - '0'], len = pass_out_count(c) * 8;
    else if (nm == "count") b = &c->ncount, len = pass_out_count(c) * 4;
    else if (nm == "store.counts" && c->has_store) b = &c->counts, len = c->num_sc * 4;
    else if (nm == "store.offsets" && c->has_store) b = &c->offsets, len = (c->num_sc + 1) * 8;
    else if (nm == "store.blob" && c->has_store) b = &c->blob, len = c->blob_bytes;
    else if (nm == "full.offsets" && c->has_full) b = &c->full_off, len = (c->full_n + 1) * 8;
    else if (nm == "sym.jacc") b = &c->sym[1], len = c->sym_e_local * (c->sym_e_kernel >= 2 ? 4 : 1) * c->sp.cj * 8;
    else if (nm == "sym.jcnt") b = &c->sym[2], len = c->sym_e_local * c->sp.cj * 4;
    else if (nm == "sym.ejcl") b = &c->sym[3], len = c->sym_e_local * 4;
    else if (nm == "sym.esc") b = &c->sym[4], len = c->sym_e_local * 4;
    else if (nm == "full.neighbors" && c->has_full) b = &c->full_nbr, len = c->full_pairs * 4;
    else if (nm.rfind("orig.", 0) == 0 && c->orig.valid) {
        const std::string f = nm.substr(5);
        Slot& o = c->orig;
        if (f == "x") b = &o.x;
        else if (f == "y") b = &o.y;
        else if (f == "z") b = &o.z;
        else if (f == "h") b = &o.h;
        else if (Field* fl = o.find(f)) b = &fl->data;
        len = o.n * 8;
    } else if (c->sorted.valid && (b = sorted_array(c, name))) len = c->sorted.n * 8;
    if (!b || (len && len > b->bytes)) return set_error(c, SFCNL_INPUT_ERROR, "device_array: no such array: " + nm);
    *ptr = b->p;
    if (bytes) *bytes = len;
    return 0;
}

}  // extern "C"
