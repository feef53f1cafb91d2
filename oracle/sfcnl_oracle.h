/* TEST INFRASTRUCTURE ONLY — the CPU restatement of the reference algorithm for
 * the compressed-neighbor-list hot path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * Parity pinning: checked against the reference's own golden vectors (codec
 * Table I, size laws, Hilbert bijection/adjacency; tests/test_oracle_golden.py)
 * and against the compiled, unmodified reference (oracle/_ref/libsfcnl_ref.so)
 * on identical inputs (tests/test_oracle_vs_ref.py, tests/golden/make_golden.py).
 *
 * Status codes mirror the reference exceptions: 0 ok, 1 InputError,
 * 2 BuildError, 3 DecodeError (byte offset via orc_last_error), 4 other.
 */
#ifndef SFCNL_ORACLE_H
#define SFCNL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(uint64_t* byte_offset);

int orc_make_uniform(uint64_t n, double density, double target, const int* per, double h_jitter,
                     uint64_t seed, double* x, double* y, double* z, double* h, double* m,
                     double* q, double* box6);
int orc_make_evrard(uint64_t n, double target, int constant_h, const int* per, uint64_t seed,
                    double* x, double* y, double* z, double* h, double* m, double* q,
                    double* box6);

int orc_hilbert_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint64_t* key);
int orc_hilbert_decode(uint64_t key, int bits, uint32_t* xyz);
int orc_sort_by_sfc(uint64_t n, const double* x, const double* y, const double* z,
                    const double* box6, const int* per, int bits, uint64_t* keys, uint32_t* perm);

/* Octree as parallel node arrays (OctreeNode field order). */
typedef struct orc_tree orc_tree;
int orc_build_octree(uint64_t n, const uint64_t* keys, int bits, uint32_t bucket, orc_tree** out);
uint64_t orc_octree_size(const orc_tree* t);
void orc_octree_nodes(const orc_tree* t, uint64_t* key_first, uint64_t* key_last,
                      uint32_t* pbegin, uint32_t* pend, int32_t* first_child, uint8_t* depth);
int orc_node_geometry(const orc_tree* t, const double* x, const double* y, const double* z,
                      const double* h, double* lo, double* hi, double* radius);
void orc_octree_free(orc_tree* t);

typedef struct orc_store orc_store;
int orc_build_store(uint64_t n, const double* x, const double* y, const double* z,
                    const double* h, const double* box6, const int* per, int bits,
                    uint64_t num_nodes, const uint64_t* key_first, const uint64_t* key_last,
                    const uint32_t* pbegin, const uint32_t* pend, const int32_t* first_child,
                    uint32_t ci, uint32_t cj, int w, int mode, int compress, double scale,
                    orc_store** out);
void orc_store_info(const orc_store* s, uint64_t* num_sc, uint64_t* blob_size);
void orc_store_copy(const orc_store* s, uint32_t* counts, uint64_t* offsets, uint8_t* blob);
void orc_store_free(orc_store* s);

int orc_codec_encode(const uint32_t* idx, uint64_t count, int w, uint8_t* out, uint64_t cap,
                     uint64_t* len);
int orc_codec_decode_into(const uint8_t* data, uint64_t size, uint32_t count, int w,
                          uint32_t* out, uint64_t* consumed);

/* kernel: 0 count, 1 SPH density ("m"), 2 LJ, 3 LJ+Coulomb ("q"). Double precision,
 * reference summation order. outs: 1 or 4 arrays of n. */
int orc_reduce(int kernel, uint64_t n, const double* x, const double* y, const double* z,
               const double* h, const double* m, const double* q, const double* box6,
               const int* per, uint32_t ci, uint32_t cj, int w, int mode, int compress,
               double scale, uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
               const uint8_t* blob, uint64_t blob_size, double query_scale, double eps,
               double sigma, double ck, double** outs, uint32_t* ncount);

/* ---- domain decomposition test helpers ----------------------
 * Node geometry from particles [p0, p1) only (lo/hi 3 per node, maxh 1 per node). */
int orc_node_geometry_range(uint64_t num_nodes, const uint32_t* pbegin, const uint32_t* pend,
                            const int32_t* first_child, const double* x, const double* y, const double* z,
                            const double* h, uint64_t p0, uint64_t p1, double* lo, double* hi, double* maxh);
/* build_neighbor_store over super-clusters [sc0, sc1) with caller node geometry
 * and global max h; the store's counts/offsets/blob are local to the range. */
int orc_build_store_range(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                          const double* box6, const int* per, uint64_t num_nodes, const uint32_t* pbegin,
                          const uint32_t* pend, const int32_t* first_child, const double* node_lo,
                          const double* node_hi, const double* node_maxh, uint32_t ci, uint32_t cj, int w,
                          int mode, int compress, double scale, uint64_t sc0, uint64_t sc1, double max_h,
                          orc_store** out);
/* Candidate j-clusters of super-clusters [sc0, sc1) (collect_candidates), as flags. */
int orc_halo_mark(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                  const double* box6, const int* per, uint64_t num_nodes, const uint32_t* pbegin,
                  const uint32_t* pend, const int32_t* first_child, const double* node_lo,
                  const double* node_hi, const double* node_maxh, uint32_t ci, uint32_t cj, int mode,
                  double scale, uint64_t sc0, uint64_t sc1, double max_h, uint8_t* jflags);
/* gather-mode reduce over a range store starting at global super-cluster sc_base;
 * outs/ncount hold the range's particles only. */
int orc_reduce_range(int kernel, uint64_t n, const double* x, const double* y, const double* z,
                     const double* h, const double* m, const double* q, const double* box6,
                     const int* per, uint32_t ci, uint32_t cj, int w, int compress, double scale,
                     uint64_t sc_base, uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
                     const uint8_t* blob, double query_scale, double eps, double sigma, double ck,
                     double** outs, uint32_t* ncount);

#ifdef __cplusplus
}
#endif
#endif
