// (3) Octree build from sorted SFC keys, node geometry, and (2) cluster geometry.
//
// Replaces build_octree (octree.cpp:9-59), compute_node_aabbs /
// compute_node_max_radius (octree.cpp:68-96) and compute_cluster_geometry
// (neighbor_build.cpp:19-38, cluster.hpp:77-90).
//
// Construction is level-synchronous instead of the reference's recursion: level d
// holds its nodes in key order; a node is internal iff count > bucket && d < bits
// (octree.cpp:14); internal nodes emit 8 children whose particle ranges come from
// binary searches over the sorted keys (the reference's lower_bound, octree.cpp:27-30).
// The reference numbers nodes in DFS allocation order: the k-th internal node in
// DFS preorder owns children [1 + 8k, 1 + 8k + 8). DFS preorder of an octree over
// disjoint key ranges is the lexicographic order of (key_first, depth), so
//   rank(X) = sum over levels d' of #internal nodes at d' with key_first < K
//           + #ancestors of X that start at K,
// computed with one binary search per level. Node arrays are therefore identical
// to the reference's, not just the leaf set.
// Geometry is computed bottom-up one level per launch (deepest first), each node
// extending its particles (leaves) or its 8 children in order, exactly as the
// reference's reverse sweep does; min/max are exact, so results are bit-equal.
// Bytes: octree ~ 8 B keys read + 32 B/node written; node geometry ~ 32 B/particle
// + 64 B/node; cluster geometry 32 B/particle read + 64 B/cluster written.
#include <algorithm>
#include <vector>

#include "ctx.hpp"
#include "scan.hpp"

namespace sfcnl_cu {
namespace {

__device__ __forceinline__ uint32_t lower_bound_keys(const uint64_t* __restrict__ keys, uint32_t lo,
                                                     uint32_t hi, uint64_t v) {
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (keys[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* __restrict__ a, uint64_t n,
                                                    uint64_t v) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_root(uint64_t* kf, uint32_t* pb, uint32_t* pe, uint32_t n) {
    kf[0] = 0, pb[0] = 0, pe[0] = n;
}

__global__ void k_flags(const uint32_t* __restrict__ pb, const uint32_t* __restrict__ pe, uint64_t m,
                        uint32_t bucket, int can_split, uint32_t* __restrict__ flag) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k < m) flag[k] = (can_split && pe[k] - pb[k] > bucket) ? 1u : 0u;
}

__global__ void k_children(int d, int bits, uint64_t m, const uint64_t* __restrict__ kf,
                           const uint32_t* __restrict__ pb, const uint32_t* __restrict__ pe,
                           const uint32_t* __restrict__ flag, const uint32_t* __restrict__ ipos,
                           const uint64_t* __restrict__ keys, uint64_t* __restrict__ ikeys,
                           uint64_t* __restrict__ ckf, uint32_t* __restrict__ cpb,
                           uint32_t* __restrict__ cpe) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= m * 8) return;
    const uint64_t k = t >> 3;
    const int c = int(t & 7);
    if (!flag[k]) return;
    const uint32_t j = ipos[k];
    if (c == 0) ikeys[j] = kf[k];
    const uint64_t span = uint64_t(1) << (3 * (bits - d - 1));
    const uint64_t cf = kf[k] + span * uint64_t(c);
    const uint32_t b = pb[k], e = pe[k];
    const uint32_t lo = c == 0 ? b : lower_bound_keys(keys, b, e, cf);
    const uint32_t hi = c == 7 ? e : lower_bound_keys(keys, b, e, cf + span);
    const uint64_t o = uint64_t(j) * 8 + c;
    ckf[o] = cf, cpb[o] = lo, cpe[o] = hi;
}

struct LevelRef {
    const uint64_t* ikeys;
    uint64_t count;
};

__global__ void k_ranks(int d, int bits, int nlev, const LevelRef* __restrict__ lev,
                        uint32_t* __restrict__ irank) {
    const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (j >= lev[d].count) return;
    const uint64_t K = lev[d].ikeys[j];
    uint64_t r = 0;
    for (int l = 0; l < nlev; ++l) {
        r += lower_bound_u64(lev[l].ikeys, lev[l].count, K);
        if (l < d) {
            const uint64_t span_mask = (uint64_t(1) << (3 * (bits - l))) - 1;
            if ((K & span_mask) == 0) ++r;
        }
    }
    irank[j] = uint32_t(r);
}

__global__ void k_write_nodes(int d, int bits, uint64_t m, const uint64_t* __restrict__ kf,
                              const uint32_t* __restrict__ pb, const uint32_t* __restrict__ pe,
                              const uint32_t* __restrict__ flag, const uint32_t* __restrict__ ipos,
                              const uint32_t* __restrict__ irank,
                              const uint32_t* __restrict__ parent_rank, Node* __restrict__ nodes,
                              uint32_t* __restrict__ level_nodes) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= m) return;
    const uint64_t idx = d == 0 ? 0 : 1 + 8 * uint64_t(parent_rank[k >> 3]) + (k & 7);
    Node nd;
    nd.key_first = kf[k];
    nd.key_last = kf[k] + (uint64_t(1) << (3 * (bits - d)));
    nd.pbegin = pb[k];
    nd.pend = pe[k];
    nd.first_child = flag[k] ? int32_t(1 + 8 * uint64_t(irank[ipos[k]])) : -1;
    nd.depth = uint8_t(d);
    nd.pad[0] = nd.pad[1] = nd.pad[2] = 0;
    nodes[idx] = nd;
    level_nodes[k] = uint32_t(idx);
}

__global__ void k_node_geo(const uint32_t* __restrict__ list, uint64_t m, const Node* __restrict__ nodes,
                           const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, const double* __restrict__ h,
                           Geo* __restrict__ geo, uint64_t p0, uint64_t p1) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= m) return;
    const uint32_t idx = list[k];
    const Node nd = nodes[idx];
    Geo g;
    geo_init(g);
    if (nd.first_child < 0) {
        // leaves see only particles [p0, p1) (a rank's partial geometry; min/max
        // combine exactly across ranks)
        const uint64_t b = nd.pbegin > p0 ? nd.pbegin : p0, e = nd.pend < p1 ? nd.pend : p1;
        for (uint64_t i = b; i < e; ++i) {
            geo_extend_pt(g, x[i], y[i], z[i]);
            g.maxh = smax(g.maxh, h[i]);
        }
    } else {
        for (int c = 0; c < 8; ++c) {
            const Geo ch = geo[nd.first_child + c];
            geo_extend(g, ch);
            g.maxh = smax(g.maxh, ch.maxh);
        }
    }
    geo[idx] = g;
}

__global__ void k_cluster_geo(uint64_t n, uint32_t width, uint64_t ncl, const double* __restrict__ x,
                              const double* __restrict__ y, const double* __restrict__ z,
                              const double* __restrict__ h, Geo* __restrict__ geo, uint64_t k0, uint64_t k1,
                              const uint8_t* __restrict__ flags) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= ncl) return;
    if ((k < k0 || k >= k1) && !(flags && flags[k])) return;  // not read by this rank
    const uint64_t b = k * width, e = tmin<uint64_t>(b + width, n);
    Geo g;
    geo_init(g);
    for (uint64_t i = b; i < e; ++i) {
        geo_extend_pt(g, x[i], y[i], z[i]);
        g.maxh = smax(g.maxh, h[i]);
    }
    geo[k] = g;
}

inline unsigned blocks_for(uint64_t m, int t = 256) { return unsigned((m + t - 1) / t); }

}  // namespace

int run_build_octree(sfcnl_cu_ctx* c, uint32_t bucket, const DistTree* dt) {
    if (bucket < 1) return set_error(c, 1, "build_octree: bucket_size must be >= 1");
    if (!c->has_order) return set_error(c, 1, "build_octree: no SFC order");
    const uint64_t n = c->order_n;
    const uint64_t n_tree = dt ? dt->n_global : n;
    if (n_tree > 0xffffffffull) return set_error(c, 1, "build_octree: more than 2^32 - 1 particles");
    const int bits = c->bits;
    stage_begin(c, kOctree);
    auto& L = c->levels;
    if (L.empty()) L.resize(1);
    SFCNL_CUDA_TRY(L[0].kf.reserve(8));
    SFCNL_CUDA_TRY(L[0].pb.reserve(4));
    SFCNL_CUDA_TRY(L[0].pe.reserve(4));
    launch(c, k_root, dim3(1), dim3(1), 0, L[0].kf.as<uint64_t>(), L[0].pb.as<uint32_t>(),
           L[0].pe.as<uint32_t>(), uint32_t(n));
    L[0].count = 1;
    // global ranges of a level: the local ones (distributed: [pb | pe] all-reduced)
    auto gpb = [&](int d) { return dt ? L[d].g.as<uint32_t>() : L[d].pb.as<uint32_t>(); };
    auto gpe = [&](int d) { return dt ? L[d].g.as<uint32_t>() + L[d].count : L[d].pe.as<uint32_t>(); };
    if (dt) {
        const uint32_t root[2] = {0u, uint32_t(n_tree)};
        SFCNL_CUDA_TRY(L[0].g.reserve(8));
        SFCNL_CUDA_TRY(cudaMemcpyAsync(L[0].g.p, root, 8, cudaMemcpyHostToDevice, c->stream));
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    int nlev = 0;
    uint64_t internal_total = 0;
    SFCNL_CUDA_TRY(c->small_host_dev.reserve(64));
    for (int d = 0;; ++d) {
        auto& lv = L[d];
        const uint64_t m = lv.count;
        SFCNL_CUDA_TRY(lv.flag.reserve(m * 4));
        SFCNL_CUDA_TRY(lv.ipos.reserve((m + 1) * 4));
        launch(c, k_flags, dim3(blocks_for(m)), dim3(256), 0, (const uint32_t*)gpb(d),
               (const uint32_t*)gpe(d), m, bucket, int(d < bits), lv.flag.as<uint32_t>());
        {
            const int rc = excl_scan(c, lv.flag.as<uint32_t>(), lv.ipos.as<uint32_t>(), m);
            if (rc) return rc;
        }
        uint32_t I = 0;
        if (int rc_rb = readback(c, &I, lv.ipos.as<uint32_t>() + m, 4)) return rc_rb;
        SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
        lv.internal = I;
        nlev = d + 1;
        if (I == 0) break;
        internal_total += I;
        if (int(L.size()) < d + 2) L.resize(d + 2);
        auto& cur = L[d];
        auto& nx = L[d + 1];
        SFCNL_CUDA_TRY(cur.ikeys.reserve(uint64_t(I) * 8));
        SFCNL_CUDA_TRY(nx.kf.reserve(uint64_t(I) * 64));
        SFCNL_CUDA_TRY(nx.pb.reserve(uint64_t(I) * 32));
        SFCNL_CUDA_TRY(nx.pe.reserve(uint64_t(I) * 32));
        nx.count = uint64_t(I) * 8;
        launch(c, k_children, dim3(blocks_for(m * 8)), dim3(256), 0, d, bits, m,
               (const uint64_t*)cur.kf.as<uint64_t>(), (const uint32_t*)cur.pb.as<uint32_t>(),
               (const uint32_t*)cur.pe.as<uint32_t>(), (const uint32_t*)cur.flag.as<uint32_t>(),
               (const uint32_t*)cur.ipos.as<uint32_t>(), (const uint64_t*)c->keys.as<uint64_t>(),
               cur.ikeys.as<uint64_t>(), nx.kf.as<uint64_t>(), nx.pb.as<uint32_t>(), nx.pe.as<uint32_t>());
        SFCNL_CUDA_TRY(cudaGetLastError());
        if (dt) {  // global child bounds = SUM over ranks of the local lower bounds
            const uint64_t cnt = nx.count;
            SFCNL_CUDA_TRY(nx.g.reserve(cnt * 8));
            SFCNL_CUDA_TRY(cudaMemcpyAsync(nx.g.p, nx.pb.p, cnt * 4, cudaMemcpyDeviceToDevice, c->stream));
            SFCNL_CUDA_TRY(cudaMemcpyAsync(nx.g.as<uint32_t>() + cnt, nx.pe.p, cnt * 4, cudaMemcpyDeviceToDevice,
                                           c->stream));
            SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
            if (dt->fn(dt->user, nx.g.as<uint32_t>(), cnt * 2))
                return set_error(c, SFCNL_CUDA_ERROR, "build_octree: all-reduce callback failed");
        }
    }
    // DFS-preorder ranks of internal nodes.
    std::vector<LevelRef> refs(nlev);
    for (int d = 0; d < nlev; ++d) refs[d] = {L[d].ikeys.as<uint64_t>(), L[d].internal};
    SFCNL_CUDA_TRY(c->level_tab.reserve(nlev * sizeof(LevelRef)));
    SFCNL_CUDA_TRY(cudaMemcpyAsync(c->level_tab.p, refs.data(), nlev * sizeof(LevelRef),
                                   cudaMemcpyHostToDevice, c->stream));
    for (int d = 0; d < nlev; ++d) {
        if (!L[d].internal) continue;
        SFCNL_CUDA_TRY(L[d].irank.reserve(L[d].internal * 4));
        launch(c, k_ranks, dim3(blocks_for(L[d].internal)), dim3(256), 0, d, bits, nlev,
               (const LevelRef*)c->level_tab.as<LevelRef>(), L[d].irank.as<uint32_t>());
    }
    const uint64_t total = 1 + 8 * internal_total;
    SFCNL_CUDA_TRY(c->nodes.reserve(total * sizeof(Node)));
    SFCNL_CUDA_TRY(c->level_nodes.reserve(total * 4));
    c->level_off.assign(nlev + 1, 0);
    for (int d = 0; d < nlev; ++d) c->level_off[d + 1] = c->level_off[d] + L[d].count;
    for (int d = 0; d < nlev; ++d) {
        launch(c, k_write_nodes, dim3(blocks_for(L[d].count)), dim3(256), 0, d, bits, L[d].count,
               (const uint64_t*)L[d].kf.as<uint64_t>(), (const uint32_t*)gpb(d),
               (const uint32_t*)gpe(d), (const uint32_t*)L[d].flag.as<uint32_t>(),
               (const uint32_t*)L[d].ipos.as<uint32_t>(), (const uint32_t*)L[d].irank.as<uint32_t>(),
               (const uint32_t*)(d ? L[d - 1].irank.as<uint32_t>() : nullptr), c->nodes.as<Node>(),
               c->level_nodes.as<uint32_t>() + c->level_off[d]);
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kOctree);
    c->num_nodes = total;
    c->tree_bits = bits;
    c->tree_n = n_tree;
    c->has_tree = true;
    drop_external(c);
    return 0;
}

int run_tree_levels_from_nodes(sfcnl_cu_ctx* c, const std::vector<uint8_t>& depth) {
    int maxd = 0;
    for (uint8_t d : depth) maxd = std::max<int>(maxd, d);
    c->level_off.assign(maxd + 2, 0);
    for (uint8_t d : depth) c->level_off[d + 1]++;
    for (int d = 0; d <= maxd; ++d) c->level_off[d + 1] += c->level_off[d];
    std::vector<uint32_t> list(depth.size());
    std::vector<uint64_t> cur(c->level_off.begin(), c->level_off.end() - 1);
    for (size_t k = 0; k < depth.size(); ++k) list[cur[depth[k]]++] = uint32_t(k);
    SFCNL_CUDA_TRY(c->level_nodes.reserve(list.size() * 4));
    SFCNL_CUDA_TRY(cudaMemcpyAsync(c->level_nodes.p, list.data(), list.size() * 4,
                                   cudaMemcpyHostToDevice, c->stream));
    SFCNL_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return 0;
}

int run_node_geometry(sfcnl_cu_ctx* c, uint64_t p0, uint64_t p1) {
    if (!c->has_tree) return set_error(c, 1, "node geometry: no octree");
    if (!c->sorted.valid || c->sorted.n != c->tree_n)
        return set_error(c, 2, "build_neighbor_store: octree/particle-set mismatch");
    SFCNL_CUDA_TRY(c->node_geo.reserve(c->num_nodes * sizeof(Geo)));
    stage_begin(c, kNodeGeo);
    const int nlev = int(c->level_off.size()) - 1;
    for (int d = nlev - 1; d >= 0; --d) {
        const uint64_t m = c->level_off[d + 1] - c->level_off[d];
        if (!m) continue;
        launch(c, k_node_geo, dim3(blocks_for(m, 128)), dim3(128), 0,
               (const uint32_t*)(c->level_nodes.as<uint32_t>() + c->level_off[d]), m,
               (const Node*)c->nodes.as<Node>(), c->sorted.x.as<const double>(),
               c->sorted.y.as<const double>(), c->sorted.z.as<const double>(),
               c->sorted.h.as<const double>(), c->node_geo.as<Geo>(), p0, p1);
    }
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kNodeGeo);
    return 0;
}

int run_cluster_geometry(sfcnl_cu_ctx* c, uint32_t ci, uint32_t cj, uint64_t p0, uint64_t p1,
                         const uint8_t* jflags) {
    const uint64_t n = c->sorted.n;
    const uint64_t ni = (n + ci - 1) / ci, nj = (n + cj - 1) / cj;
    SFCNL_CUDA_TRY(c->igeo.reserve(std::max<uint64_t>(ni, 1) * sizeof(Geo)));
    SFCNL_CUDA_TRY(c->jgeo.reserve(std::max<uint64_t>(nj, 1) * sizeof(Geo)));
    if (!n) return 0;
    if (p1 > n) p1 = n;
    c->clgeo_whole = p0 == 0 && p1 == n && !jflags;
    stage_begin(c, kClusterGeo);
    // i-clusters: the range (plus the flagged halo when the array doubles as jgeo)
    launch(c, k_cluster_geo, dim3(blocks_for(ni)), dim3(256), 0, n, ci, ni, c->sorted.x.as<const double>(),
           c->sorted.y.as<const double>(), c->sorted.z.as<const double>(), c->sorted.h.as<const double>(),
           c->igeo.as<Geo>(), p0 / ci, (p1 + ci - 1) / ci, cj == ci ? jflags : (const uint8_t*)nullptr);
    if (cj != ci)
        launch(c, k_cluster_geo, dim3(blocks_for(nj)), dim3(256), 0, n, cj, nj, c->sorted.x.as<const double>(),
               c->sorted.y.as<const double>(), c->sorted.z.as<const double>(),
               c->sorted.h.as<const double>(), c->jgeo.as<Geo>(), p0 / cj, (p1 + cj - 1) / cj, jflags);
    SFCNL_CUDA_TRY(cudaGetLastError());
    stage_end(c, kClusterGeo);
    return 0;
}

}  // namespace sfcnl_cu
