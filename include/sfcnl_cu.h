/*
 * sfcnl_cu.h — C-ABI of the B200-native (sm_100a) compressed clustered neighbor
 * list: SFC keygen + sort + permute, cornerstone-style octree, cluster geometry,
 * warp-cooperative traversal + interaction masks, nibble-codec encode, and the
 * in-kernel-decoding neighborhood pass.
 *
 * This is the drop-in boundary for the reference's build-and-query path
 * (reference = /root/reference/proj, C++20, CPU only). Each entry point names the
 * reference interface it replaces. Plain pointers and sizes only; no exceptions
 * and no C++ types cross it. The C++ drop-in (include/sfcnl/*.hpp, the
 * reference's public API re-implemented over this ABI) maps the status codes
 * back to the reference exception types:
 *
 *   SFCNL_OK 0, SFCNL_INPUT_ERROR 1 -> sfcnl::InputError (core.hpp:18),
 *   SFCNL_BUILD_ERROR 2 -> sfcnl::BuildError (core.hpp:23),
 *   SFCNL_DECODE_ERROR 3 -> sfcnl::DecodeError{byte_offset} (core.hpp:28),
 *   SFCNL_CUDA_ERROR 4 -> std::runtime_error.
 *
 * Memory model: a context owns one CUDA stream on one device and the device
 * copies of everything it computes. "set_*" calls copy host arrays in,
 * "get_*" calls copy results out; every call is synchronous at return unless
 * its comment says otherwise. All host pointers may be pageable or pinned; the
 * array arguments of set_* / get_* may also be device pointers (copies use
 * cudaMemcpyDefault), which keeps a multi-rank step device-resident.
 */
#ifndef SFCNL_CU_H
#define SFCNL_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFCNL_OK 0
#define SFCNL_INPUT_ERROR 1
#define SFCNL_BUILD_ERROR 2
#define SFCNL_DECODE_ERROR 3
#define SFCNL_CUDA_ERROR 4

typedef struct sfcnl_cu_ctx sfcnl_cu_ctx;

/* SimulationBox (core.hpp:50-74). */
typedef struct {
    double lo[3];
    double hi[3];
    int32_t periodic[3];
} sfcnl_box;

/* OctreeNode (octree.hpp:11-21), identical 32-byte layout. */
typedef struct {
    uint64_t key_first;
    uint64_t key_last;
    uint32_t particle_begin;
    uint32_t particle_end;
    int32_t first_child;
    uint8_t depth;
    uint8_t pad_[3];
} sfcnl_node;

/* BuildParams + ClusterParams (neighbor_store.hpp:18-29, cluster.hpp:12-29).
 * mode: 0 gather, 1 symmetric. sc_size is fixed at 64 (cluster.hpp:9). */
typedef struct {
    uint32_t ci;
    uint32_t cj;
    int32_t w;
    int32_t mode;
    int32_t compress;
    double build_radius_scale;
} sfcnl_build_params;

/* Built-in pair kernels (builtin_kernels.hpp:24-95). */
#define SFCNL_KERNEL_COUNT 0      /* CountKernel: 1 output "count"            */
#define SFCNL_KERNEL_DENSITY 1    /* SphDensityKernel: 1 output "rho", in "m" */
#define SFCNL_KERNEL_LJ 2         /* LjKernel<Real,false>: fx, fy, fz, energy */
#define SFCNL_KERNEL_LJ_COULOMB 3 /* LjKernel<Real,true>: + Coulomb on "q"    */

/* precision: 0 = fp64, bitwise equal to reduce<double> (reference summation
 *                 order, no FMA);
 *            1 = mixed (fp32 pair math on SC-relative coordinates, exact fp64
 *                 cutoff decisions via a guard band, fp64 lane combine);
 *                 neighbor_count exact, values within 1e-5 of reduce<double>. */
typedef struct {
    int32_t kernel;
    int32_t precision;
    double query_scale;
    double epsilon;
    double sigma;
    double coulomb_k;
} sfcnl_pass_params;

/* ---- context ------------------------------------------------------------ */
int sfcnl_cu_ctx_create(int device, sfcnl_cu_ctx** out);
void sfcnl_cu_ctx_destroy(sfcnl_cu_ctx* ctx);
/* Message of the last failed call on this context (or of a failed create when
 * ctx == NULL); *byte_offset receives DecodeError::byte_offset. */
const char* sfcnl_cu_last_error(sfcnl_cu_ctx* ctx, uint64_t* byte_offset);
/* cudaStream_t of the context (for event timing by the caller). */
void* sfcnl_cu_stream(sfcnl_cu_ctx* ctx);
int sfcnl_cu_synchronize(sfcnl_cu_ctx* ctx);
/* Number of kernels this context has launched so far. */
uint64_t sfcnl_cu_launch_count(sfcnl_cu_ctx* ctx);
/* Per-stage device times (ms) of the most recent calls, in the order
 * keygen, sort, permute, octree, node_geometry, cluster_geometry, build, encode,
 * pass; returns the number written (<= cap). Enabled by sfcnl_cu_set_timing. */
int sfcnl_cu_set_timing(sfcnl_cu_ctx* ctx, int enabled);
int sfcnl_cu_stage_times(sfcnl_cu_ctx* ctx, double* ms, int cap);

/* ---- particles ------------------------------------------------------------
 * ParticleSet (core.hpp:168-198) in original (unsorted) order. Fields are named
 * payload arrays ("m", "q", ...). Replaces nothing by itself: it is the upload
 * half of every reference call that takes `const ParticleSet&`. */
int sfcnl_cu_set_particles(sfcnl_cu_ctx* ctx, uint64_t n, const double* x, const double* y,
                           const double* z, const double* h, const sfcnl_box* box);
int sfcnl_cu_set_field(sfcnl_cu_ctx* ctx, const char* name, const double* values);
/* Same, for a set that is ALREADY in SFC order (the `sorted` argument of
 * build_neighbor_store / reduce): marks it as the sorted slot directly. */
int sfcnl_cu_set_sorted_particles(sfcnl_cu_ctx* ctx, uint64_t n, const double* x,
                                  const double* y, const double* z, const double* h,
                                  const sfcnl_box* box);
int sfcnl_cu_set_sorted_field(sfcnl_cu_ctx* ctx, const char* name, const double* values);

/* ---- (1) SFC keys + stable radix sort ---------------------------------------
 * Replaces sort_by_sfc (hilbert.hpp:126, hilbert.cpp:8-26): keys = sfc_key of every
 * particle (hilbert.hpp:110-113), perm = stable ascending order. Results stay on
 * the device; sfcnl_cu_get_order downloads them. */
int sfcnl_cu_sort_by_sfc(sfcnl_cu_ctx* ctx, int bits);
int sfcnl_cu_get_order(sfcnl_cu_ctx* ctx, uint64_t* keys, uint32_t* perm);
/* Upload an SfcOrder computed elsewhere (keys ascending, perm a permutation). */
int sfcnl_cu_set_order(sfcnl_cu_ctx* ctx, uint64_t n, const uint64_t* keys, const uint32_t* perm,
                       int bits);

/* Replaces apply_sfc_order (hilbert.hpp:129, hilbert.cpp:28-44): gathers x,y,z,h
 * and every field into the sorted slot. */
int sfcnl_cu_apply_order(sfcnl_cu_ctx* ctx);
/* Download one sorted array: "x","y","z","h" or a field name. */
int sfcnl_cu_get_sorted(sfcnl_cu_ctx* ctx, const char* name, double* out);

/* ---- (3) octree --------------------------------------------------------------
 * Replaces build_octree (octree.hpp:51, octree.cpp:43-59) on the current keys:
 * same node set and the same node numbering (parent before children, children
 * contiguous, DFS allocation order). */
int sfcnl_cu_build_octree(sfcnl_cu_ctx* ctx, uint32_t bucket_size, uint64_t* num_nodes);
int sfcnl_cu_get_octree(sfcnl_cu_ctx* ctx, sfcnl_node* nodes);
/* Upload a caller-provided Octree (e.g. the `tree` argument of build_neighbor_store). */
int sfcnl_cu_set_octree(sfcnl_cu_ctx* ctx, uint64_t num_nodes, const sfcnl_node* nodes, int bits,
                        uint64_t n);
/* Replaces compute_node_aabbs + compute_node_max_radius (octree.hpp:57-60,
 * octree.cpp:68-96) on the sorted slot. lo/hi: 3 doubles per node; radius: 1. */
int sfcnl_cu_node_geometry(sfcnl_cu_ctx* ctx, double* lo, double* hi, double* radius);

/* ---- (2)(3)(4) list build ----------------------------------------------------
 * Replaces build_neighbor_store (neighbor_build.hpp:18-19, neighbor_build.cpp:74-184)
 * on the sorted slot and the current octree: cluster geometry, traversal, masks,
 * nibble-codec encode (nibble_codec.cpp:117-134). Output is byte-identical to the
 * reference NeighborStore (counts, offsets, blob). */
int sfcnl_cu_build_store(sfcnl_cu_ctx* ctx, const sfcnl_build_params* params,
                         uint64_t* num_superclusters, uint64_t* blob_bytes);
int sfcnl_cu_get_store(sfcnl_cu_ctx* ctx, uint32_t* counts, uint64_t* offsets, uint8_t* blob);
/* Upload a NeighborStore (neighbor_store.hpp:44-59) for a later reduce. */
int sfcnl_cu_set_store(sfcnl_cu_ctx* ctx, const sfcnl_build_params* params, uint64_t n,
                       uint64_t num_superclusters, const uint32_t* counts,
                       const uint64_t* offsets, const uint8_t* blob, uint64_t blob_bytes);

/* ---- (5) neighborhood pass ---------------------------------------------------
 * Replaces reduce<Real,K> (reduce.hpp:38-231) for the built-in kernels, gather
 * and symmetric stores, on the sorted slot and the current store. outs: 1 or 4
 * host arrays of n doubles (NULL = keep on device); count: n uint32 (nullable). */
int sfcnl_cu_reduce(sfcnl_cu_ctx* ctx, const sfcnl_pass_params* params, double* const* outs,
                    uint32_t* neighbor_count);

/* ---- (5a) device view for user pair kernels ------------------------------------
 * reduce<Real, K> with a user kernel (make_pair_kernel / BasicPairKernel,
 * pair_kernel.hpp:60-91; reduce.hpp:38-231) runs a header-only CUDA kernel in the
 * caller's own CUDA translation unit (include/sfcnl/gpu_pair_kernel.cuh) over the
 * context's device state: the sorted particle set, its fields and the store set by
 * sfcnl_cu_set_sorted_field / sfcnl_cu_set_store. Pointers stay valid until the next
 * call that changes that state. box_len[d] is the periodic length of axis d, 0 on
 * open axes (the reference's box_len, reduce.hpp:80-81). */
typedef struct {
    uint64_t n;
    uint64_t num_sc;
    uint32_t ci;
    uint32_t cj;
    int32_t w;
    int32_t mode;
    int32_t compress;
    double box_len[3];
    const double* x;
    const double* y;
    const double* z;
    const double* h;
    const uint32_t* counts;
    const uint64_t* offsets;
    const uint8_t* blob;
    uint64_t blob_bytes;
    void* stream;
} sfcnl_cu_device_view;
int sfcnl_cu_get_device_view(sfcnl_cu_ctx* ctx, sfcnl_cu_device_view* out);
/* device pointer of a field of the sorted slot (set by sfcnl_cu_set_sorted_field) */
int sfcnl_cu_sorted_field_ptr(sfcnl_cu_ctx* ctx, const char* name, const double** out);

/* ---- (5b) full Verlet list baseline -------------------------
 * The classic per-particle CSR list the paper measures the compressed list
 * against (baselines.hpp:27-38 FullVerletList, :42-44 build_full_list, :47-129
 * reduce_full). build_full_list derives it on the device from the current
 * whole-range GATHER store: for every i the j != i with
 * |minimage(x_i - x_j)|^2 <= (build_scale h_i)^2 (periodic_delta, fp64), ascending
 * j -- the same list as build_full_list(sorted, box, build_scale, gather) for any
 * build_scale <= the store's build radius scale. num_pairs = offsets[n].
 * get_full_list: offsets u64[n + 1], neighbors u32[num_pairs]. set_full_list
 * uploads a list built elsewhere (mode 0 gather, 1 symmetric). reduce_full
 * replaces reduce_full<Real,K>: precision 0 is bit-equal to reduce_full<double>
 * (ascending j, thread per i); precision 1 evaluates the same pairs warp-per-i in
 * fp64 with a tree sum. outs/count as in sfcnl_cu_reduce. */
int sfcnl_cu_build_full_list(sfcnl_cu_ctx* ctx, double build_scale, uint64_t* num_pairs);
int sfcnl_cu_get_full_list(sfcnl_cu_ctx* ctx, uint64_t* offsets, uint32_t* neighbors);
int sfcnl_cu_set_full_list(sfcnl_cu_ctx* ctx, uint64_t n, int mode, double build_scale,
                           const uint64_t* offsets, const uint32_t* neighbors, uint64_t num_pairs);
int sfcnl_cu_reduce_full(sfcnl_cu_ctx* ctx, const sfcnl_pass_params* params, double* const* outs,
                         uint32_t* neighbor_count);

/* Numerator of cluster_overhead (bench.cpp:93-122) for the current gather store:
 * the pair slots the pass evaluates, sum over entries and set mask bits of
 * |i-cluster| * |j-cluster|. overhead = slots / true directed pairs. */
int sfcnl_cu_cluster_slots(sfcnl_cu_ctx* ctx, uint64_t* slots);

/* ---- (6) SFC domain decomposition -----------------------------
 * The reference is single-process; these entry points let one process per GPU
 * own a contiguous range of super-clusters of the GLOBAL sorted order while the
 * store it builds is byte-identical to the corresponding slice of the
 * single-domain store (neighbor_build.cpp:74-184 restricted to sc in
 * [sc_begin, sc_end)). Particles outside the range but inside the halo must be
 * present in the sorted slot at their global index.
 *
 * build_store_range: as build_store over super-clusters [sc_begin, sc_end)
 * (clamped to the particle count). max_h > 0 overrides the local max(h) used by
 * the traversal (pass the global all-reduced max so every rank prunes alike).
 * The resulting store's counts/offsets/blob are local to the range; reduce then
 * writes outputs for particles [64*sc_begin, min(n, 64*sc_end)) only. Gather
 * mode only for ranges other than the whole set. */
int sfcnl_cu_build_store_range(sfcnl_cu_ctx* ctx, const sfcnl_build_params* params, uint64_t sc_begin,
                               uint64_t sc_end, double max_h, uint64_t* num_superclusters,
                               uint64_t* blob_bytes);
/* Input slot from a DEVICE row-major [n, ncols] record array whose columns are
 * x, y, z, h and then the ncols - 4 named fields (the layout an all-to-all of
 * particle rows delivers); same effect as set_particles + set_field. */
int sfcnl_cu_set_particle_records(sfcnl_cu_ctx* ctx, uint64_t n, const double* records, int ncols,
                                  const char* const* fields, const sfcnl_box* box);
/* Allocate the sorted slot for n particles with the named extra fields (contents
 * undefined) so ranks can fill it piecewise with write_sorted. Invalidates the
 * store. */
int sfcnl_cu_alloc_sorted(sfcnl_cu_ctx* ctx, uint64_t n, const sfcnl_box* box, const char* const* fields,
                          int nfields);
/* Copy count doubles into / out of sorted array `name` ("x","y","z","h" or a
 * field) at element offset. *_on_device: the other pointer is device memory. */
int sfcnl_cu_write_sorted(sfcnl_cu_ctx* ctx, const char* name, uint64_t offset, uint64_t count,
                          const double* src, int src_on_device);
int sfcnl_cu_read_sorted(sfcnl_cu_ctx* ctx, const char* name, uint64_t offset, uint64_t count, double* dst,
                         int dst_on_device);
/* Read a sub-range of the current SfcOrder (keys and/or perm, nullable). */
int sfcnl_cu_read_order(sfcnl_cu_ctx* ctx, uint64_t offset, uint64_t count, uint64_t* keys, uint32_t* perm,
                        int dst_on_device);
/* Install globally sorted keys (e.g. all-gathered from the ranks) as the order
 * build_octree consumes; perm is left undefined (apply_order must not follow). */
int sfcnl_cu_set_keys(sfcnl_cu_ctx* ctx, uint64_t n, const uint64_t* keys, int src_on_device, int bits);
/* apply_sfc_order (hilbert.cpp:28-44) into elements [offset, offset + n) of an
 * allocated sorted slot (alloc_sorted) that holds every field of the input slot:
 * a rank places its owned, locally sorted particles at their global positions. */
int sfcnl_cu_apply_order_into(sfcnl_cu_ctx* ctx, uint64_t offset);
/* compute_node_aabbs / compute_node_max_radius (octree.cpp:68-96) over particles
 * [p_begin, p_end) only: every rank computes the partial geometry of the global
 * octree from its own particles; an element-wise min (lo) / max (hi, maxh)
 * all-reduce of the "node_geo" device array (8 doubles per node: lo[3], hi[3],
 * maxh, pad) then yields the exact global geometry. Marks the array as
 * caller-managed: halo_mark / build_store_range use it as is. */
int sfcnl_cu_node_geometry_range(sfcnl_cu_ctx* ctx, uint64_t p_begin, uint64_t p_end);
/* Flag (u8 per global j-cluster, device array "halo_flags") every j-cluster that
 * build_store_range(sc_begin, sc_end) will read: the candidate clusters of
 * collect_candidates (neighbor_build.cpp:43-65) for each super-cluster of the
 * range. Needs positions/h of the range's own particles, the global octree and
 * its (all-reduced) node geometry. A following build_store_range over the same
 * range computes cluster geometry only for the range and the flagged halo. */
int sfcnl_cu_halo_mark(sfcnl_cu_ctx* ctx, const sfcnl_build_params* params, uint64_t sc_begin,
                       uint64_t sc_end, uint64_t* num_jclusters);
/* Symmetric stores over a super-cluster range (the reference's ordered j-side commit,
 * reduce.hpp:186-218, across ranks). sym_range_entries: the j-side accumulators of the
 * range's entries (reference order, fp64) -> device arrays "sym.jacc" (entries x outputs x
 * cj doubles), "sym.jcnt" (entries x cj), "sym.ejcl" (global j-cluster), "sym.esc"
 * (global super-cluster). sym_range_final: DEVICE arrays of the entries received from
 * earlier ranks (same layouts, in global entry order) are prepended to the local ones
 * and every particle of the range folds them around its own i side; outputs / count
 * as in sfcnl_cu_reduce for the range's particles. Bit-equal to the single-domain
 * reduce<double> on a symmetric store. */
int sfcnl_cu_sym_range_entries(sfcnl_cu_ctx* ctx, const sfcnl_pass_params* params, uint64_t* num_entries);
int sfcnl_cu_sym_range_final(sfcnl_cu_ctx* ctx, const sfcnl_pass_params* params, uint64_t num_remote,
                             const double* jacc, const uint32_t* jcnt, const uint32_t* ejcl,
                             const uint32_t* esc, double* const* outs, uint32_t* neighbor_count);
/* ---- (6b) O(N/P) decomposition: local index space, distributed octree ---------
 * Per rank memory proportional to its own particles plus its halo:
 *   key_hist          radix-select splitter: for each of nq boundaries, the number of
 *                     LOCAL sorted keys (the current SfcOrder) in each of the 65536
 *                     buckets [prefix[q] + b << shift, prefix[q] + (b + 1) << shift);
 *                     hist is a DEVICE int64 array of nq x 65536 (sum it over ranks).
 *   merge_runs        owner placement: the n received rows are nruns runs (host
 *                     run_bounds[nruns + 1]), each sorted by (key, global id); rows are
 *                     written to out in (key, run) order = the global stable order.
 *                     cols / out: HOST arrays of ncols DEVICE column pointers.
 *   build_octree_dist build_octree (octree.cpp:9-59) of the GLOBAL key multiset whose
 *                     local part is the current SfcOrder: per level the child bounds
 *                     (local lower bounds) are summed over ranks by fn (in-place SUM of
 *                     count u32 on the device, on the context's stream). Identical node
 *                     arrays on every rank (reference numbering), global particle ranges.
 *   leaf_boxes        per node (6 doubles lo[3], hi[3], DEVICE num_nodes x 6): the box of
 *                     the rank's particles of every LEAF overlapping [p_begin, p_end)
 *                     (x/y/z: DEVICE owned columns, element g - p_begin); other nodes empty.
 *   domain_boxes      the boxes of nbox equal chunks of the owned particles (nbox x 6).
 *   halo_select       owner side of the halo: flags[q * n_owned_clusters + k] = 1 when
 *                     owned cluster k (cj particles from p_begin) overlaps a leaf whose
 *                     box is within `reach` (periodic aabb_dist_sq) of one of rank q's
 *                     nbox domain boxes (DEVICE nranks x nbox x 6); the rank's own row is
 *                     left zero. Conservative: every leaf any super-cluster of rank q can
 *                     accept (collect_candidates, neighbor_build.cpp:43-65) is selected.
 *   pack_clusters     rows (DEVICE, nclusters*cj x ncols, row-major) of the listed owned
 *                     clusters (global ids) from the owned columns; tail slots past p_end
 *                     are NaN.
 *   dd_place          local index space: the sorted slot (alloc_sorted(n_local)) receives
 *                     the owned columns and the halo rows at local cluster lpos[c] (DEVICE
 *                     u32 per global cluster); padding clusters (lc2g == ~0) are NaN.
 *                     Also writes lc2g (local cluster -> global cluster).
 *   dd_localize       the global octree's particle ranges mapped to the local index space
 *                     (g -> lpos[g / cj] * cj + (present ? g % cj : 0)), and the maps that
 *                     the range build (local clusters -> global ids in the encoded list)
 *                     and the passes (decoded global ids -> local clusters) use.
 *   dd_lc2g           lc2g[lpos[c]] = c for every present global cluster c, ~0 elsewhere.
 *   dd_clear          back to the single-domain index space. */
typedef int (*sfcnl_allreduce_u32)(void* user, uint32_t* device_data, uint64_t count);
int sfcnl_cu_key_hist(sfcnl_cu_ctx* ctx, uint32_t nq, const uint64_t* prefix, int shift, int64_t* hist);
int sfcnl_cu_merge_runs(sfcnl_cu_ctx* ctx, uint64_t n, uint32_t ncols, const double* const* cols,
                        const uint64_t* keys, uint32_t nruns, const uint64_t* run_bounds, double* const* out);
int sfcnl_cu_build_octree_dist(sfcnl_cu_ctx* ctx, uint32_t bucket, uint64_t n_global, sfcnl_allreduce_u32 fn,
                               void* user, uint64_t* num_nodes);
int sfcnl_cu_leaf_boxes(sfcnl_cu_ctx* ctx, uint64_t p_begin, uint64_t p_end, const double* x, const double* y,
                        const double* z, double* boxes);
int sfcnl_cu_domain_boxes(sfcnl_cu_ctx* ctx, uint64_t n_owned, const double* x, const double* y, const double* z,
                          uint32_t nbox, double* boxes);
int sfcnl_cu_halo_select(sfcnl_cu_ctx* ctx, uint64_t p_begin, uint64_t p_end, uint32_t cj,
                         const double* leaf_boxes, uint32_t nranks, uint32_t self_rank, uint32_t nbox,
                         const double* domain_boxes, double reach, uint8_t* flags);
int sfcnl_cu_pack_clusters(sfcnl_cu_ctx* ctx, uint64_t p_begin, uint64_t p_end, uint32_t cj,
                           const uint32_t* clusters, uint64_t nclusters, uint32_t ncols,
                           const double* const* cols, double* rows);
int sfcnl_cu_dd_place(sfcnl_cu_ctx* ctx, uint64_t n_global, uint64_t p_begin, uint64_t p_end, uint32_t cj,
                      const uint32_t* lpos, uint64_t n_local, uint32_t ncols, const double* const* owned_cols,
                      const uint32_t* halo_clusters, uint64_t nhalo, const double* halo_rows, uint32_t* lc2g);
int sfcnl_cu_dd_localize(sfcnl_cu_ctx* ctx, uint32_t cj, const uint32_t* lpos, const uint8_t* present,
                         uint64_t n_global_clusters, const uint32_t* lc2g);
int sfcnl_cu_dd_lc2g(sfcnl_cu_ctx* ctx, uint64_t n_global_clusters, const uint32_t* lpos, const uint8_t* present,
                     uint32_t* lc2g, uint64_t n_local_clusters);
int sfcnl_cu_dd_clear(sfcnl_cu_ctx* ctx);
/* Device bytes currently allocated by the context (every internal buffer). */
int sfcnl_cu_memory_bytes(sfcnl_cu_ctx* ctx, uint64_t* bytes);

/* Device pointer + byte length of an internal array for zero-copy collectives:
 * "x","y","z","h", sorted fields by name, "keys","perm","nodes","node_geo",
 * "halo_flags","out0".."out3","count", the input slot "orig.x".."orig.h" and
 * "orig.<field>", the store "store.counts","store.offsets","store.blob", the full
 * list "full.offsets","full.neighbors", the symmetric range entries "sym.jacc",
 * "sym.jcnt","sym.ejcl","sym.esc".
 * Valid until the next call that resizes it. */
int sfcnl_cu_device_array(sfcnl_cu_ctx* ctx, const char* name, void** ptr, uint64_t* bytes);

/* ---- host-side codec (no device work) ----------------------------------------
 * codec::encode / codec::decode_into (nibble_codec.hpp:54-60), used by the C++
 * drop-in and by the parity tests. encode: *len receives the byte length; bytes
 * are written only when *len <= cap. */
int sfcnl_codec_encode(const uint32_t* indices, uint64_t count, int w, uint8_t* out,
                       uint64_t cap, uint64_t* len);
int sfcnl_codec_decode_into(const uint8_t* data, uint64_t size, uint32_t count, int w,
                            uint32_t* out, uint64_t* consumed);
/* hilbert_encode / hilbert_decode (hilbert.hpp:66-90), host-side. */
int sfcnl_hilbert_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint64_t* key);
int sfcnl_hilbert_decode(uint64_t key, int bits, uint32_t* xyz);
const char* sfcnl_last_host_error(uint64_t* byte_offset);

/* ---- fixtures ---------------------------------------------------------------
 * make_uniform / make_evrard (generators.hpp:34-35): host generators, seeded,
 * byte-identical to the reference's. box6 = lo[3], hi[3]. */
int sfcnl_make_uniform(uint64_t n, double density, double target, const int32_t* periodic,
                       double h_jitter, uint64_t seed, double* x, double* y, double* z,
                       double* h, double* m, double* q, double* box6);
int sfcnl_make_evrard(uint64_t n, double target, int32_t constant_h, const int32_t* periodic,
                      uint64_t seed, double* x, double* y, double* z, double* h, double* m,
                      double* q, double* box6);

#ifdef __cplusplus
}
#endif
#endif /* SFCNL_CU_H */
