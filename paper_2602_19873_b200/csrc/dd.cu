// O(N/P) SFC domain decomposition: the per-rank device side of
// paper_2602_19873_b200/distributed.py (include/sfcnl_cu.h section (6b)).
//
// The reference is single-process (parallel_for over super-clusters,
// neighbor_build.cpp:109, reduce.hpp:217-220). A rank owns the particles [p0, p1) of the
// GLOBAL SFC order (p0, p1 multiples of 64, so its super-clusters are global ones) and
// holds, in a LOCAL index space, only those plus its halo:
//
//   local = [halo clusters below p0][NaN padding to a multiple of 64][owned][halo above]
//
// in ascending global order. The map global cluster -> local cluster (lpos) is monotone
// and cluster-granular, so every octree node's particle range maps to a contiguous
// local range, the leaf -> j-cluster rule of collect_candidates (neighbor_build.cpp:
// 53-60, including the "shared with the previous leaf" de-duplication) is unchanged,
// and the rank's super-clusters are whole local super-clusters. The encoder writes
// global cluster ids (lc2g) so the store bytes equal the single-domain slice; the pass
// decoders map the stored global ids back (lpos). NaN padding is invisible: boxes use
// std::min/max semantics (NaN loses), fp32/fp64 pair tests with NaN are false.
//
// Kernels here: radix-select histogram (splitter), k-way merge of the received runs,
// per-leaf boxes of the owned particles, domain chunk boxes, owner-side halo selection,
// cluster packing, local placement and tree localisation. The distributed octree itself
// is octree.cu (run_build_octree with a DistTree).
#include <algorithm>
#include <vector>

#include "ctx.hpp"

namespace sfcnl_cu {
namespace {

constexpr int kHistBins = 65536;
#define kInf __longlong_as_double(0x7ff0000000000000LL)

__device__ __forceinline__ uint64_t lb_u64(const uint64_t* __restrict__ a, uint64_t n, uint64_t v) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint64_t ub_u64(const uint64_t* __restrict__ a, uint64_t n, uint64_t v) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// hist[q][b] = #keys in [prefix[q] + b << shift, prefix[q] + (b + 1) << shift)
__global__ void k_key_hist(const uint64_t* __restrict__ keys, uint64_t n, uint32_t nq,
                           const uint64_t* __restrict__ prefix, int shift, long long* __restrict__ hist) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(nq) * kHistBins) return;
    const uint32_t q = uint32_t(t / kHistBins), b = uint32_t(t % kHistBins);
    const uint64_t base = prefix[q];
    const uint64_t step = uint64_t(1) << shift;
    // bounds past 2^64 are past every key (keys < 2^63)
    auto bound = [&](uint64_t k) -> uint64_t {
        const unsigned __int128 v = (unsigned __int128)base + (unsigned __int128)k * step;
        return v >> 64 ? n : lb_u64(keys, n, uint64_t(v));
    };
    hist[t] = (long long)(bound(uint64_t(b) + 1) - bound(b));
}

// Row r of run s goes to position (r - start_s) + #(run q < s: key <= k) + #(run q > s: key < k)
__global__ void k_merge_runs(uint64_t n, uint32_t ncols, const double* const* __restrict__ cols,
                             const uint64_t* __restrict__ keys, uint32_t nruns, const uint64_t* __restrict__ bounds,
                             double* const* __restrict__ out) {
    const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    uint32_t s = 0;
    while (s + 1 < nruns && bounds[s + 1] <= r) ++s;
    const uint64_t k = keys[r];
    uint64_t dst = r - bounds[s];
    for (uint32_t q = 0; q < nruns; ++q) {
        if (q == s) continue;
        const uint64_t b = bounds[q], e = bounds[q + 1];
        dst += q < s ? ub_u64(keys + b, e - b, k) : lb_u64(keys + b, e - b, k);
    }
    for (uint32_t c = 0; c < ncols; ++c) out[c][dst] = cols[c][r];
}

// Leaves overlapping [p0, p1): box of their particles in that range (x[g - p0]).
__global__ void k_leaf_boxes(uint64_t num_nodes, const Node* __restrict__ nodes, uint64_t p0, uint64_t p1,
                             const double* __restrict__ x, const double* __restrict__ y,
                             const double* __restrict__ z, double* __restrict__ boxes) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= num_nodes) return;
    const Node nd = nodes[k];
    double lo[3] = {kInf, kInf, kInf}, hi[3] = {-kInf, -kInf, -kInf};
    if (nd.first_child < 0) {
        const uint64_t b = nd.pbegin > p0 ? nd.pbegin : p0, e = nd.pend < p1 ? nd.pend : p1;
        for (uint64_t g = b; g < e; ++g) {
            const double v[3] = {x[g - p0], y[g - p0], z[g - p0]};
#pragma unroll
            for (int d = 0; d < 3; ++d) lo[d] = smin(lo[d], v[d]), hi[d] = smax(hi[d], v[d]);
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) boxes[k * 6 + d] = lo[d], boxes[k * 6 + 3 + d] = hi[d];
}

// Box of each of nbox chunks (whole super-clusters) of the owned particles (block per chunk).
__global__ void k_domain_boxes(uint64_t n, const double* __restrict__ x, const double* __restrict__ y,
                               const double* __restrict__ z, uint32_t nbox, double* __restrict__ boxes) {
    __shared__ double red[6][256];
    // chunks of whole super-clusters: every super-cluster box lies inside one chunk box
    const uint64_t m = ((n + nbox - 1) / nbox + 63) / 64 * 64;
    const uint64_t b = uint64_t(blockIdx.x) * m, e = b + m < n ? b + m : n;
    double lo[3] = {kInf, kInf, kInf}, hi[3] = {-kInf, -kInf, -kInf};
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const double v[3] = {x[i], y[i], z[i]};
#pragma unroll
        for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], v[d]), hi[d] = fmax(hi[d], v[d]);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) red[d][threadIdx.x] = lo[d], red[3 + d][threadIdx.x] = hi[d];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                red[d][threadIdx.x] = fmin(red[d][threadIdx.x], red[d][threadIdx.x + s]);
                red[3 + d][threadIdx.x] = fmax(red[3 + d][threadIdx.x], red[3 + d][threadIdx.x + s]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) boxes[blockIdx.x * 6 + threadIdx.x] = red[threadIdx.x][0];
}

// Owner side of the halo (thread per node): a leaf overlapping the owned range whose
// box is within `reach` of one of rank q's domain boxes flags its owned clusters for q.
__global__ void k_halo_select(uint64_t num_nodes, const Node* __restrict__ nodes, uint64_t p0, uint64_t p1,
                              uint32_t cj, const double* __restrict__ leaf_boxes, uint32_t nranks, uint32_t self,
                              uint32_t nbox, const double* __restrict__ dboxes, Box box, double reach2,
                              uint8_t* __restrict__ flags, uint64_t nown_cl) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= num_nodes) return;
    const Node nd = nodes[k];
    if (nd.first_child >= 0 || nd.pend <= p0 || nd.pbegin >= p1 || nd.pend <= nd.pbegin) return;
    Geo lb;
#pragma unroll
    for (int d = 0; d < 3; ++d) lb.lo[d] = leaf_boxes[k * 6 + d], lb.hi[d] = leaf_boxes[k * 6 + 3 + d];
    lb.maxh = 0.0, lb.pad = 0.0;
    const uint64_t b = nd.pbegin > p0 ? nd.pbegin : p0, e = nd.pend < p1 ? nd.pend : p1;
    const uint64_t c0 = b / cj - p0 / cj, c1 = (e - 1) / cj - p0 / cj;
    for (uint32_t q = 0; q < nranks; ++q) {
        if (q == self) continue;
        bool near = false;
        for (uint32_t t = 0; t < nbox && !near; ++t) {
            Geo db;
            const double* s = dboxes + (uint64_t(q) * nbox + t) * 6;
#pragma unroll
            for (int d = 0; d < 3; ++d) db.lo[d] = s[d], db.hi[d] = s[3 + d];
            db.maxh = 0.0, db.pad = 0.0;
            near = !(aabb_dist_sq(lb, db, box) > reach2);
        }
        if (near)
            for (uint64_t c = c0; c <= c1; ++c) flags[uint64_t(q) * nown_cl + c] = 1;
    }
}

__global__ void k_pack_clusters(uint64_t p0, uint64_t p1, uint32_t cj, const uint32_t* __restrict__ ids,
                                uint64_t nids, uint32_t ncols, const double* const* __restrict__ cols,
                                double* __restrict__ rows) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= nids * cj) return;
    const uint64_t g = uint64_t(ids[t / cj]) * cj + t % cj;
    const bool ok = g >= p0 && g < p1;
    for (uint32_t c = 0; c < ncols; ++c) rows[t * ncols + c] = ok ? cols[c][g - p0] : __longlong_as_double(0x7ff8000000000000LL);
}

// Local placement: thread per local particle slot of the owned block and the halo rows;
// padding slots (lc2g == ~0) NaN. ncols columns: x, y, z, h, fields (sorted slot order).
__global__ void k_dd_place_owned(uint64_t p0, uint64_t p1, uint32_t cj, const uint32_t* __restrict__ lpos,
                                 uint32_t ncols, const double* const* __restrict__ owned, double* const* __restrict__ out) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= p1 - p0) return;
    const uint64_t g = p0 + t;
    const uint64_t l = uint64_t(lpos[g / cj]) * cj + g % cj;
    for (uint32_t c = 0; c < ncols; ++c) out[c][l] = owned[c][t];
}

__global__ void k_dd_place_halo(uint64_t n_global, uint32_t cj, const uint32_t* __restrict__ lpos,
                                const uint32_t* __restrict__ ids, uint64_t nids, uint32_t ncols,
                                const double* __restrict__ rows, double* const* __restrict__ out) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= nids * cj) return;
    const uint64_t c = ids[t / cj], g = c * cj + t % cj;
    if (g >= n_global) return;
    const uint64_t l = uint64_t(lpos[c]) * cj + t % cj;
    for (uint32_t k = 0; k < ncols; ++k) out[k][l] = rows[t * ncols + k];
}

__global__ void k_dd_fill(uint64_t n_local, uint32_t cj, const uint32_t* __restrict__ lc2g, uint32_t ncols,
                          double* const* __restrict__ out) {
    const uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (l >= n_local) return;
    if (lc2g[l / cj] != 0xffffffffu) return;
    for (uint32_t k = 0; k < ncols; ++k) out[k][l] = __longlong_as_double(0x7ff8000000000000LL);
}

// lc2g from lpos over the present global clusters
__global__ void k_dd_lc2g(uint64_t ngc, const uint32_t* __restrict__ lpos, const uint8_t* __restrict__ present,
                          uint32_t* __restrict__ lc2g) {
    const uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (c < ngc && present[c]) lc2g[lpos[c]] = uint32_t(c);
}

__global__ void k_dd_localize(uint64_t num_nodes, Node* __restrict__ nodes, uint32_t cj, uint64_t ngc,
                              const uint32_t* __restrict__ lpos, const uint8_t* __restrict__ present) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= num_nodes) return;
    Node nd = nodes[k];
    auto map = [&](uint64_t g) -> uint32_t {
        const uint64_t c = g / cj;
        if (c >= ngc) return uint32_t(uint64_t(lpos[ngc]) * cj);
        return uint32_t(uint64_t(lpos[c]) * cj + (present[c] ? g % cj : 0));
    };
    const uint32_t b = map(nd.pbegin), e = map(nd.pend);
    nd.pbegin = b, nd.pend = e > b ? e : b;
    nodes[k] = nd;
}

inline unsigned blocks(uint64_t m, int t = 256) { return unsigned((m + t - 1) / t); }

}  // namespace

uint64_t& dbuf_total_bytes() {
    static uint64_t total = 0;
    return total;
}

}  // namespace sfcnl_cu

using namespace sfcnl_cu;

namespace {
// host array of device pointers -> device table in c->dd_tab at byte offset `off`
int put_ptrs(sfcnl_cu_ctx* c, const void* const* host, uint32_t n, size_t off) {
    SFCNL_CUDA_TRY(cudaMemcpyAsync(c->dd_tab.as<uint8_t>() + off, host, n * sizeof(void*), cudaMemcpyHostToDevice,
                                   c->stream));
    return 0;
}
int finish_dd(sfcnl_cu_ctx* c) {
    SFCNL_CUDA_TRY(cudaGetLastError());
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return 0;
}
}  // namespace

extern "C" {

int sfcnl_cu_key_hist(sfcnl_cu_ctx* c, uint32_t nq, const uint64_t* prefix, int shift, int64_t* hist) {
    if (!c || !c->has_order) return c ? set_error(c, SFCNL_INPUT_ERROR, "key_hist: no SFC order") : SFCNL_INPUT_ERROR;
    if (shift < 0 || shift > 48) return set_error(c, SFCNL_INPUT_ERROR, "key_hist: bad shift");
    if (nq)
        launch(c, k_key_hist, dim3(blocks(uint64_t(nq) * kHistBins)), dim3(256), 0, c->keys.as<const uint64_t>(),
               c->order_n, nq, prefix, shift, reinterpret_cast<long long*>(hist));
    return finish_dd(c);
}

int sfcnl_cu_merge_runs(sfcnl_cu_ctx* c, uint64_t n, uint32_t ncols, const double* const* cols, const uint64_t* keys,
                        uint32_t nruns, const uint64_t* run_bounds, double* const* out) {
    if (!c) return SFCNL_INPUT_ERROR;
    if (ncols > 32 || nruns == 0 || nruns > 4096) return set_error(c, SFCNL_INPUT_ERROR, "merge_runs: bad arguments");
    SFCNL_CUDA_TRY(c->dd_tab.reserve(2 * 32 * sizeof(void*) + (nruns + 1) * 8));
    if (int rc = put_ptrs(c, reinterpret_cast<const void* const*>(cols), ncols, 0)) return rc;
    if (int rc = put_ptrs(c, reinterpret_cast<const void* const*>(out), ncols, 32 * sizeof(void*))) return rc;
    uint64_t* dbounds = reinterpret_cast<uint64_t*>(c->dd_tab.as<uint8_t>() + 64 * sizeof(void*));
    SFCNL_CUDA_TRY(cudaMemcpyAsync(dbounds, run_bounds, (nruns + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    if (n)
        launch(c, k_merge_runs, dim3(blocks(n)), dim3(256), 0, n, ncols,
               reinterpret_cast<const double* const*>(c->dd_tab.as<uint8_t>()), keys, nruns, (const uint64_t*)dbounds,
               reinterpret_cast<double* const*>(c->dd_tab.as<uint8_t>() + 32 * sizeof(void*)));
    return finish_dd(c);
}

int sfcnl_cu_build_octree_dist(sfcnl_cu_ctx* c, uint32_t bucket, uint64_t n_global, sfcnl_allreduce_u32 fn,
                               void* user, uint64_t* num_nodes) {
    if (!c) return SFCNL_INPUT_ERROR;
    if (!fn) return set_error(c, SFCNL_INPUT_ERROR, "build_octree_dist: null all-reduce");
    const DistTree dt{n_global, fn, user};
    if (int rc = run_build_octree(c, bucket, &dt)) return rc;
    if (num_nodes) *num_nodes = c->num_nodes;
    return finish_dd(c);
}

int sfcnl_cu_leaf_boxes(sfcnl_cu_ctx* c, uint64_t p0, uint64_t p1, const double* x, const double* y, const double* z,
                        double* boxes) {
    if (!c || !c->has_tree) return c ? set_error(c, SFCNL_INPUT_ERROR, "leaf_boxes: no octree") : SFCNL_INPUT_ERROR;
    if (c->num_nodes)
        launch(c, k_leaf_boxes, dim3(blocks(c->num_nodes)), dim3(256), 0, c->num_nodes, c->nodes.as<const Node>(), p0,
               p1, x, y, z, boxes);
    return finish_dd(c);
}

int sfcnl_cu_domain_boxes(sfcnl_cu_ctx* c, uint64_t n, const double* x, const double* y, const double* z, uint32_t nbox,
                          double* boxes) {
    if (!c || nbox == 0) return c ? set_error(c, SFCNL_INPUT_ERROR, "domain_boxes: nbox must be > 0") : SFCNL_INPUT_ERROR;
    launch(c, k_domain_boxes, dim3(nbox), dim3(256), 0, n, x, y, z, nbox, boxes);
    return finish_dd(c);
}

int sfcnl_cu_halo_select(sfcnl_cu_ctx* c, uint64_t p0, uint64_t p1, uint32_t cj, const double* leaf_boxes,
                         uint32_t nranks, uint32_t self_rank, uint32_t nbox, const double* domain_boxes, double reach,
                         uint8_t* flags) {
    if (!c || !c->has_tree) return c ? set_error(c, SFCNL_INPUT_ERROR, "halo_select: no octree") : SFCNL_INPUT_ERROR;
    if (cj == 0 || p0 % cj) return set_error(c, SFCNL_INPUT_ERROR, "halo_select: range not cluster aligned");
    const uint64_t nown_cl = (p1 - p0 + cj - 1) / cj;
    if (nranks && nown_cl) SFCNL_CUDA_TRY(cudaMemsetAsync(flags, 0, uint64_t(nranks) * nown_cl, c->stream));
    const double reach2 = reach * reach;  // conservative bound (no exactness needed)
    Box box = c->sorted.valid ? c->sorted.box : c->orig.box;
    if (c->num_nodes && nranks)
        launch(c, k_halo_select, dim3(blocks(c->num_nodes)), dim3(256), 0, c->num_nodes, c->nodes.as<const Node>(), p0,
               p1, cj, leaf_boxes, nranks, self_rank, nbox, domain_boxes, box, reach2, flags, nown_cl);
    return finish_dd(c);
}

int sfcnl_cu_pack_clusters(sfcnl_cu_ctx* c, uint64_t p0, uint64_t p1, uint32_t cj, const uint32_t* ids, uint64_t nids,
                           uint32_t ncols, const double* const* cols, double* rows) {
    if (!c) return SFCNL_INPUT_ERROR;
    if (ncols > 32) return set_error(c, SFCNL_INPUT_ERROR, "pack_clusters: too many columns");
    SFCNL_CUDA_TRY(c->dd_tab.reserve(2 * 32 * sizeof(void*) + 8));
    if (int rc = put_ptrs(c, reinterpret_cast<const void* const*>(cols), ncols, 0)) return rc;
    if (nids)
        launch(c, k_pack_clusters, dim3(blocks(nids * cj)), dim3(256), 0, p0, p1, cj, ids, nids, ncols,
               reinterpret_cast<const double* const*>(c->dd_tab.as<uint8_t>()), rows);
    return finish_dd(c);
}

int sfcnl_cu_dd_place(sfcnl_cu_ctx* c, uint64_t n_global, uint64_t p0, uint64_t p1, uint32_t cj, const uint32_t* lpos,
                      uint64_t n_local, uint32_t ncols, const double* const* owned_cols, const uint32_t* halo_ids,
                      uint64_t nhalo, const double* halo_rows, uint32_t* lc2g) {
    if (!c) return SFCNL_INPUT_ERROR;
    Slot& s = c->sorted;
    if (!s.valid || s.n != n_local || ncols != 4 + s.fields.size())
        return set_error(c, SFCNL_INPUT_ERROR, "dd_place: allocate the sorted slot (alloc_sorted) for n_local first");
    SFCNL_CUDA_TRY(c->dd_tab.reserve(2 * 32 * sizeof(void*) + 8));
    std::vector<const void*> dst = {s.x.p, s.y.p, s.z.p, s.h.p};
    for (auto& f : s.fields) dst.push_back(f.data.p);
    if (int rc = put_ptrs(c, reinterpret_cast<const void* const*>(owned_cols), ncols, 0)) return rc;
    if (int rc = put_ptrs(c, dst.data(), ncols, 32 * sizeof(void*))) return rc;
    auto* tab_in = reinterpret_cast<const double* const*>(c->dd_tab.as<uint8_t>());
    auto* tab_out = reinterpret_cast<double* const*>(c->dd_tab.as<uint8_t>() + 32 * sizeof(void*));
    if (p1 > p0)
        launch(c, k_dd_place_owned, dim3(blocks(p1 - p0)), dim3(256), 0, p0, p1, cj, lpos, ncols, tab_in, tab_out);
    if (nhalo)
        launch(c, k_dd_place_halo, dim3(blocks(nhalo * cj)), dim3(256), 0, n_global, cj, lpos, halo_ids, nhalo, ncols,
               halo_rows, tab_out);
    if (n_local) launch(c, k_dd_fill, dim3(blocks(n_local)), dim3(256), 0, n_local, cj, (const uint32_t*)lc2g, ncols, tab_out);
    c->has_store = false;
    ++c->store_gen;
    return finish_dd(c);
}

int sfcnl_cu_dd_localize(sfcnl_cu_ctx* c, uint32_t cj, const uint32_t* lpos, const uint8_t* present, uint64_t ngc,
                         const uint32_t* lc2g) {
    if (!c || !c->has_tree) return c ? set_error(c, SFCNL_INPUT_ERROR, "dd_localize: no octree") : SFCNL_INPUT_ERROR;
    if (!c->sorted.valid) return set_error(c, SFCNL_INPUT_ERROR, "dd_localize: no local particles");
    if (c->num_nodes)
        launch(c, k_dd_localize, dim3(blocks(c->num_nodes)), dim3(256), 0, c->num_nodes, c->nodes.as<Node>(), cj, ngc,
               lpos, present);
    c->tree_n = c->sorted.n;
    c->dd_lc2g = lc2g;
    c->dd_g2l = lpos;
    c->has_store = false;
    ++c->store_gen;
    drop_external(c);
    return finish_dd(c);
}

int sfcnl_cu_dd_clear(sfcnl_cu_ctx* c) {
    if (!c) return SFCNL_INPUT_ERROR;
    c->dd_lc2g = nullptr;
    c->dd_g2l = nullptr;
    return 0;
}

int sfcnl_cu_memory_bytes(sfcnl_cu_ctx* c, uint64_t* bytes) {
    if (!c || !bytes) return SFCNL_INPUT_ERROR;
    *bytes = dbuf_total_bytes();
    return 0;
}

// lc2g for the present clusters (used by dd_place's padding fill): exposed through
// dd_place's caller in distributed.py via torch; kept here for the kernel set.
int sfcnl_cu_dd_lc2g(sfcnl_cu_ctx* c, uint64_t ngc, const uint32_t* lpos, const uint8_t* present, uint32_t* lc2g,
                     uint64_t n_local_clusters) {
    if (!c) return SFCNL_INPUT_ERROR;
    if (n_local_clusters) SFCNL_CUDA_TRY(cudaMemsetAsync(lc2g, 0xff, n_local_clusters * 4, c->stream));
    if (ngc) launch(c, k_dd_lc2g, dim3(blocks(ngc)), dim3(256), 0, ngc, lpos, present, lc2g);
    return finish_dd(c);
}

}  // extern "C"
