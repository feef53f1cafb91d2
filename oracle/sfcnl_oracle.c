/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See sfcnl_oracle.h for who may use it and how it is pinned.
 * Compiled with -ffp-contract=off, like the reference (proj/src/CMakeLists.txt:14),
 * so every floating-point expression below rounds exactly as the reference's does.
 * Reference paths are relative to /root/reference/proj.
 */
#include "sfcnl_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_msg[256];
static _Thread_local uint64_t g_off;

static int fail(int code, const char* msg, uint64_t off) {
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    g_off = off;
    return code;
}

const char* orc_last_error(uint64_t* byte_offset) {
    if (byte_offset) *byte_offset = g_off;
    return g_msg;
}

/* std::min / std::max semantics (first argument wins ties). */
static inline double dmin(double a, double b) { return (b < a) ? b : a; }
static inline double dmax(double a, double b) { return (a < b) ? b : a; }

/* ---------------------------------------------------------------- generators
 * generators.cpp:12 canonical() over std::mt19937_64 (standard MT19937-64). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

static double canonical(mt64* r) { return (double)(mt64_next(r) >> 11) * 0x1.0p-53; }

static const double kPi = 3.141592653589793; /* std::numbers::pi_v<double> */

/* generators.cpp:21-45 */
int orc_make_uniform(uint64_t n, double density, double target, const int* per, double h_jitter,
                     uint64_t seed, double* x, double* y, double* z, double* h, double* m,
                     double* q, double* box6) {
    (void)per;
    if (n < 1) return fail(1, "make_uniform: n must be >= 1", 0);
    if (!(h_jitter >= 0) || h_jitter >= 1) return fail(1, "make_uniform: h_jitter must be in [0, 1)", 0);
    if (!(target > 0) || !(density > 0)) return fail(1, "uniform_h_for_target: positive inputs required", 0);
    const double side = cbrt((double)n / density);
    const double h0 = cbrt(3.0 * target / (4.0 * kPi * density));
    mt64* r = (mt64*)malloc(sizeof(mt64));
    mt64_seed(r, seed);
    for (uint64_t i = 0; i < n; ++i) {
        x[i] = canonical(r) * side;
        y[i] = canonical(r) * side;
        z[i] = canonical(r) * side;
        h[i] = h_jitter > 0 ? h0 * (1.0 + h_jitter * (2.0 * canonical(r) - 1.0)) : h0;
    }
    free(r);
    for (uint64_t i = 0; i < n; ++i) {
        if (m) m[i] = 1.0;
        if (q) q[i] = (i % 2 == 0) ? 1.0 : -1.0;
    }
    for (int d = 0; d < 3; ++d) box6[d] = 0.0, box6[3 + d] = side;
    return 0;
}

/* generators.cpp:47-82 */
int orc_make_evrard(uint64_t n, double target, int constant_h, const int* per, uint64_t seed,
                    double* x, double* y, double* z, double* h, double* m, double* q,
                    double* box6) {
    (void)per;
    if (n < 1) return fail(1, "make_evrard: n must be >= 1", 0);
    const double R = 1.0, margin = 1.1 * R;
    const double alpha = cbrt(3.0 * target / (4.0 * kPi));
    const double mean_r = 2.0 / 3.0 * R;
    mt64* r = (mt64*)malloc(sizeof(mt64));
    mt64_seed(r, seed);
    for (uint64_t i = 0; i < n; ++i) {
        const double rad = R * sqrt(canonical(r));
        const double cos_t = 1.0 - 2.0 * canonical(r);
        const double sin_t = sqrt(dmax(0.0, 1.0 - cos_t * cos_t));
        const double phi = 2.0 * kPi * canonical(r);
        x[i] = rad * sin_t * cos(phi);
        y[i] = rad * sin_t * sin(phi);
        z[i] = rad * cos_t;
        const double r_for_h = constant_h ? mean_r : rad;
        const double spacing = cbrt(2.0 * kPi * R * R * r_for_h / (double)n);
        h[i] = alpha * spacing;
    }
    free(r);
    for (uint64_t i = 0; i < n; ++i) {
        if (m) m[i] = 1.0 / (double)n;
        if (q) q[i] = (i % 2 == 0) ? 1.0 : -1.0;
    }
    for (int d = 0; d < 3; ++d) box6[d] = -margin, box6[3 + d] = margin;
    return 0;
}

/* ---------------------------------------------------------------- Hilbert keys
 * hilbert.hpp:20-38 (Skilling transpose), :66-77 (interleave, X[0] most significant),
 * :94-107 (grid coords), :110-113 (sfc_key), core.hpp:65-73 (wrap). */
static void axes_to_transpose(uint32_t X[3], int bits) {
    for (uint32_t q = 1u << (bits - 1); q > 1; q >>= 1) {
        const uint32_t p = q - 1;
        for (int i = 0; i < 3; ++i) {
            if (X[i] & q) {
                X[0] ^= p;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & p;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];
    X[2] ^= X[1];
    uint32_t t = 0;
    for (uint32_t q = 1u << (bits - 1); q > 1; q >>= 1)
        if (X[2] & q) t ^= q - 1;
    X[0] ^= t, X[1] ^= t, X[2] ^= t;
}

/* hilbert.hpp:40-57 */
static void transpose_to_axes(uint32_t X[3], int bits) {
    const uint32_t n = 2u << (bits - 1);
    uint32_t t = X[2] >> 1;
    X[2] ^= X[1];
    X[1] ^= X[0];
    X[0] ^= t;
    for (uint32_t q = 2; q != n; q <<= 1) {
        const uint32_t p = q - 1;
        for (int i = 2; i >= 0; --i) {
            if (X[i] & q) {
                X[0] ^= p;
            } else {
                t = (X[0] ^ X[i]) & p;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
}

int orc_hilbert_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint64_t* key) {
    if (bits < 1 || bits > 21) return fail(1, "bits per dimension must be in [1, 21]", 0);
    const uint32_t lim = (1u << bits) - 1;
    if (ix > lim || iy > lim || iz > lim) return fail(1, "grid coordinate out of range", 0);
    uint32_t X[3] = {ix, iy, iz};
    axes_to_transpose(X, bits);
    uint64_t k = 0;
    for (int b = bits - 1; b >= 0; --b)
        for (int i = 0; i < 3; ++i) k = (k << 1) | ((X[i] >> b) & 1u);
    *key = k;
    return 0;
}

int orc_hilbert_decode(uint64_t key, int bits, uint32_t* xyz) {
    if (bits < 1 || bits > 21) return fail(1, "bits per dimension must be in [1, 21]", 0);
    if (bits < 21 && key >= (1ULL << (3 * bits))) return fail(1, "Hilbert key out of range", 0);
    uint32_t X[3] = {0, 0, 0};
    for (int b = bits - 1; b >= 0; --b)
        for (int i = 0; i < 3; ++i) X[i] |= (uint32_t)((key >> (3 * b + (2 - i))) & 1u) << b;
    transpose_to_axes(X, bits);
    xyz[0] = X[0], xyz[1] = X[1], xyz[2] = X[2];
    return 0;
}

typedef struct {
    double lo[3], hi[3];
    int per[3];
} box_t;

static box_t mkbox(const double* box6, const int* per) {
    box_t b;
    for (int d = 0; d < 3; ++d) b.lo[d] = box6[d], b.hi[d] = box6[3 + d], b.per[d] = per[d] != 0;
    return b;
}

static double blen(const box_t* b, int d) { return b->hi[d] - b->lo[d]; }

static int sfc_key(const double p0[3], const box_t* b, int bits, uint64_t* key) {
    double p[3] = {p0[0], p0[1], p0[2]};
    for (int d = 0; d < 3; ++d) { /* SimulationBox::wrap */
        if (!b->per[d]) continue;
        const double L = blen(b, d);
        p[d] -= L * floor((p[d] - b->lo[d]) / L);
        if (p[d] >= b->hi[d]) p[d] = b->lo[d];
    }
    const double cells = (double)(1ULL << bits);
    uint32_t g[3];
    for (int d = 0; d < 3; ++d) { /* grid_coords */
        if (!isfinite(p[d])) return fail(1, "grid_coords: non-finite coordinate", 0);
        double f = (p[d] - b->lo[d]) / blen(b, d) * cells;
        if (f < 0) f = 0;
        double c = floor(f);
        if (c > cells - 1) c = cells - 1;
        g[d] = (uint32_t)c;
    }
    return orc_hilbert_encode(g[0], g[1], g[2], bits, key);
}

/* hilbert.cpp:8-26: keys, then a stable sort of the identity permutation by key.
 * Restated as an LSD radix sort (stable by construction) over 16-bit digits. */
int orc_sort_by_sfc(uint64_t n, const double* x, const double* y, const double* z,
                    const double* box6, const int* per, int bits, uint64_t* keys, uint32_t* perm) {
    if (bits < 1 || bits > 21) return fail(1, "bits per dimension must be in [1, 21]", 0);
    const box_t b = mkbox(box6, per);
    uint64_t* k0 = (uint64_t*)malloc((n + 1) * 8);
    uint64_t* k1 = (uint64_t*)malloc((n + 1) * 8);
    uint32_t* p0 = (uint32_t*)malloc((n + 1) * 4);
    uint32_t* p1 = (uint32_t*)malloc((n + 1) * 4);
    for (uint64_t i = 0; i < n; ++i) {
        const double p[3] = {x[i], y[i], z[i]};
        const int rc = sfc_key(p, &b, bits, &k0[i]);
        if (rc) {
            free(k0), free(k1), free(p0), free(p1);
            return rc;
        }
        p0[i] = (uint32_t)i;
    }
    static uint64_t cnt[65536];
    for (int shift = 0; shift < 64; shift += 16) {
        memset(cnt, 0, sizeof cnt);
        for (uint64_t i = 0; i < n; ++i) cnt[(k0[i] >> shift) & 0xffff]++;
        uint64_t s = 0;
        for (int d = 0; d < 65536; ++d) {
            const uint64_t c = cnt[d];
            cnt[d] = s;
            s += c;
        }
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t dst = cnt[(k0[i] >> shift) & 0xffff]++;
            k1[dst] = k0[i];
            p1[dst] = p0[i];
        }
        uint64_t* tk = k0; k0 = k1; k1 = tk;
        uint32_t* tp = p0; p0 = p1; p1 = tp;
    }
    memcpy(keys, k0, n * 8);
    memcpy(perm, p0, n * 4);
    free(k0), free(k1), free(p0), free(p1);
    return 0;
}

/* ---------------------------------------------------------------- octree
 * octree.cpp:9-59: top-down subdivision; children allocated contiguously when a
 * node is subdivided; recursion in child order (parent-before-children layout). */
typedef struct {
    uint64_t key_first, key_last;
    uint32_t pbegin, pend;
    int32_t first_child;
    uint8_t depth;
} node_t;

struct orc_tree {
    node_t* nodes;
    uint64_t size, cap;
    int bits;
    uint64_t n;
};

static void tree_push(struct orc_tree* t, node_t nd) {
    if (t->size == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 64;
        t->nodes = (node_t*)realloc(t->nodes, t->cap * sizeof(node_t));
    }
    t->nodes[t->size++] = nd;
}

static uint64_t lower_bound_u64(const uint64_t* a, uint64_t lo, uint64_t hi, uint64_t v) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

static void subdivide(struct orc_tree* t, uint64_t node, const uint64_t* keys, uint32_t bucket) {
    const node_t nd = t->nodes[node];
    if (nd.pend - nd.pbegin <= bucket || nd.depth >= t->bits) return;
    const int32_t first_child = (int32_t)t->size;
    t->nodes[node].first_child = first_child;
    const uint64_t span = (nd.key_last - nd.key_first) / 8;
    uint32_t child_begin = nd.pbegin;
    for (int c = 0; c < 8; ++c) {
        node_t ch;
        ch.key_first = nd.key_first + span * (uint64_t)c;
        ch.key_last = ch.key_first + span;
        ch.pbegin = child_begin;
        ch.pend = (c == 7) ? nd.pend
                           : (uint32_t)lower_bound_u64(keys, nd.pbegin, nd.pend, ch.key_last);
        ch.first_child = -1;
        ch.depth = (uint8_t)(nd.depth + 1);
        tree_push(t, ch);
        child_begin = ch.pend;
    }
    for (int c = 0; c < 8; ++c) subdivide(t, (uint64_t)first_child + c, keys, bucket);
}

int orc_build_octree(uint64_t n, const uint64_t* keys, int bits, uint32_t bucket, orc_tree** out) {
    if (bucket < 1) return fail(1, "build_octree: bucket_size must be >= 1", 0);
    struct orc_tree* t = (struct orc_tree*)calloc(1, sizeof(struct orc_tree));
    t->bits = bits;
    t->n = n;
    node_t root = {0, 1ULL << (3 * bits), 0, (uint32_t)n, -1, 0};
    tree_push(t, root);
    subdivide(t, 0, keys, bucket);
    *out = t;
    return 0;
}

uint64_t orc_octree_size(const orc_tree* t) { return t->size; }

void orc_octree_nodes(const orc_tree* t, uint64_t* key_first, uint64_t* key_last,
                      uint32_t* pbegin, uint32_t* pend, int32_t* first_child, uint8_t* depth) {
    for (uint64_t k = 0; k < t->size; ++k) {
        key_first[k] = t->nodes[k].key_first;
        key_last[k] = t->nodes[k].key_last;
        pbegin[k] = t->nodes[k].pbegin;
        pend[k] = t->nodes[k].pend;
        first_child[k] = t->nodes[k].first_child;
        depth[k] = t->nodes[k].depth;
    }
}

void orc_octree_free(orc_tree* t) {
    if (!t) return;
    free(t->nodes);
    free(t);
}

/* Aabb (core.hpp:88-113): empty = +inf/-inf; extend with std::min/std::max. */
typedef struct {
    double lo[3], hi[3];
} aabb_t;

static aabb_t aabb_empty(void) {
    aabb_t a;
    for (int d = 0; d < 3; ++d) a.lo[d] = INFINITY, a.hi[d] = -INFINITY;
    return a;
}
static int aabb_is_empty(const aabb_t* a) { return a->lo[0] > a->hi[0]; }
static void aabb_extend_pt(aabb_t* a, const double p[3]) {
    for (int d = 0; d < 3; ++d) a->lo[d] = dmin(a->lo[d], p[d]), a->hi[d] = dmax(a->hi[d], p[d]);
}
static void aabb_extend(aabb_t* a, const aabb_t* o) {
    if (aabb_is_empty(o)) return;
    aabb_extend_pt(a, o->lo);
    aabb_extend_pt(a, o->hi);
}

/* octree.cpp:68-96: reverse sweep, children before parents. */
int orc_node_geometry(const orc_tree* t, const double* x, const double* y, const double* z,
                      const double* h, double* lo, double* hi, double* radius) {
    aabb_t* boxes = (aabb_t*)malloc((t->size + 1) * sizeof(aabb_t));
    for (uint64_t k = t->size; k-- > 0;) {
        const node_t* nd = &t->nodes[k];
        boxes[k] = aabb_empty();
        radius[k] = 0.0;
        if (nd->first_child < 0) {
            for (uint32_t i = nd->pbegin; i < nd->pend; ++i) {
                const double p[3] = {x[i], y[i], z[i]};
                aabb_extend_pt(&boxes[k], p);
                radius[k] = dmax(radius[k], h[i]);
            }
        } else {
            for (int c = 0; c < 8; ++c) {
                aabb_extend(&boxes[k], &boxes[nd->first_child + c]);
                radius[k] = dmax(radius[k], radius[nd->first_child + c]);
            }
        }
        for (int d = 0; d < 3; ++d) lo[3 * k + d] = boxes[k].lo[d], hi[3 * k + d] = boxes[k].hi[d];
    }
    free(boxes);
    return 0;
}

/* octree.cpp:68-96 restricted to particles [p0, p1) (a rank's partial geometry;
 * element-wise min/max over ranks gives the global one). Arrays per node. */
int orc_node_geometry_range(uint64_t num_nodes, const uint32_t* pbegin, const uint32_t* pend,
                            const int32_t* first_child, const double* x, const double* y, const double* z,
                            const double* h, uint64_t p0, uint64_t p1, double* lo, double* hi, double* maxh) {
    for (uint64_t k = num_nodes; k-- > 0;) {
        aabb_t b = aabb_empty();
        double r = 0.0;
        if (first_child[k] < 0) {
            const uint64_t s0 = pbegin[k] > p0 ? pbegin[k] : p0, s1 = pend[k] < p1 ? pend[k] : p1;
            for (uint64_t i = s0; i < s1; ++i) {
                const double p[3] = {x[i], y[i], z[i]};
                aabb_extend_pt(&b, p);
                r = dmax(r, h[i]);
            }
        } else {
            for (int c = 0; c < 8; ++c) {
                const uint64_t ch = (uint64_t)(first_child[k] + c);
                aabb_t cb;
                for (int d = 0; d < 3; ++d) cb.lo[d] = lo[3 * ch + d], cb.hi[d] = hi[3 * ch + d];
                aabb_extend(&b, &cb);
                r = dmax(r, maxh[ch]);
            }
        }
        for (int d = 0; d < 3; ++d) lo[3 * k + d] = b.lo[d], hi[3 * k + d] = b.hi[d];
        maxh[k] = r;
    }
    return 0;
}

/* ---------------------------------------------------------------- predicates
 * core.hpp:77-85 periodic_delta, :132-135 interval_interval_gap, :152-165 aabb_dist_sq. */
static double periodic_d2(const double a[3], const double b[3], const box_t* bx, double d[3]) {
    for (int ax = 0; ax < 3; ++ax) {
        d[ax] = a[ax] - b[ax];
        if (!bx->per[ax]) continue;
        const double L = blen(bx, ax);
        d[ax] -= L * rint(d[ax] / L);
    }
    return d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
}

static double ii_gap(double alo, double ahi, double blo, double bhi) {
    const double g = dmax(alo, blo) - dmin(ahi, bhi);
    return g > 0 ? g : 0.0;
}

static double aabb_dist_sq(const aabb_t* a, const aabb_t* b, const box_t* bx) {
    if (aabb_is_empty(a) || aabb_is_empty(b)) return INFINITY;
    double s = 0;
    for (int d = 0; d < 3; ++d) {
        double g = ii_gap(a->lo[d], a->hi[d], b->lo[d], b->hi[d]);
        if (bx->per[d]) {
            const double L = blen(bx, d);
            g = dmin(g, ii_gap(a->lo[d], a->hi[d], b->lo[d] - L, b->hi[d] - L));
            g = dmin(g, ii_gap(a->lo[d], a->hi[d], b->lo[d] + L, b->hi[d] + L));
        }
        s += g * g;
    }
    return s;
}

/* ---------------------------------------------------------------- nibble codec
 * nibble_codec.cpp:56-134 (encode), :136-178 (decode_into). */
typedef struct {
    uint8_t* b;
    uint64_t len, cap;
} bytes_t;

static void bput(bytes_t* s, uint8_t v) {
    if (s->len == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 256;
        s->b = (uint8_t*)realloc(s->b, s->cap);
    }
    s->b[s->len++] = v;
}

static int nibble_count(uint64_t v) {
    int bw = 0;
    while (v) ++bw, v >>= 1;
    return (bw + 3) / 4;
}

static int codec_encode_into(const uint32_t* idx, uint64_t count, int w, bytes_t* out) {
    if (w != 32 && w != 64) return fail(1, "block width must be 32 or 64", 0);
    uint64_t prev = 0;
    uint8_t nib[64 * 9];
    for (uint64_t begin = 0; begin < count; begin += (uint64_t)w) {
        const uint64_t len = (count - begin < (uint64_t)w) ? count - begin : (uint64_t)w;
        uint64_t mask = 0;
        int ninfo = 0, ndata = 0;
        uint8_t info[64], data[64 * 8];
        for (uint64_t k = 0; k < len; ++k) {
            const uint64_t cur = idx[begin + k];
            uint64_t v;
            if (begin + k == 0) {
                v = cur + 1;
            } else {
                if (cur <= prev) return fail(1, "delta_encode: input not strictly increasing", 0);
                v = cur - prev;
            }
            prev = cur;
            if (v > 0xffffffffULL) return fail(1, "encode_block: difference exceeds 2^32 - 1", 0);
            if (v == 1) continue;
            mask |= 1ULL << k;
            if (v <= 9) {
                info[ninfo++] = (uint8_t)(v + 6);
            } else {
                const int nn = nibble_count(v);
                info[ninfo++] = (uint8_t)(nn - 1);
                for (int p = nn - 1; p >= 0; --p) data[ndata++] = (uint8_t)((v >> (4 * p)) & 0xf);
            }
        }
        for (int byte = 0; byte < w / 8; ++byte) bput(out, (uint8_t)((mask >> (8 * byte)) & 0xff));
        int nn = 0;
        for (int i = 0; i < ninfo; ++i) nib[nn++] = info[i];
        for (int i = 0; i < ndata; ++i) nib[nn++] = data[i];
        for (int i = 0; i < nn; i += 2)
            bput(out, (uint8_t)((nib[i] & 0xf) | ((i + 1 < nn ? nib[i + 1] : 0) << 4)));
    }
    return 0;
}

int orc_codec_encode(const uint32_t* idx, uint64_t count, int w, uint8_t* out, uint64_t cap,
                     uint64_t* len) {
    bytes_t b = {0, 0, 0};
    const int rc = codec_encode_into(idx, count, w, &b);
    if (rc == 0) {
        *len = b.len;
        if (b.len <= cap && b.len) memcpy(out, b.b, b.len);
    }
    free(b.b);
    return rc;
}

int orc_codec_decode_into(const uint8_t* data, uint64_t size, uint32_t count, int w,
                          uint32_t* out, uint64_t* consumed) {
    if (w != 32 && w != 64) return fail(1, "block width must be 32 or 64", 0);
    uint64_t pos = 0;
    int half = 0;
    uint64_t running = 0;
    uint32_t produced = 0;
#define TAKE(dst)                                                              \
    do {                                                                       \
        if (pos >= size) return fail(3, "truncated nibble stream", pos);       \
        if (half) { half = 0; dst = (uint8_t)(data[pos++] >> 4); }             \
        else { half = 1; dst = (uint8_t)(data[pos] & 0xf); }                   \
    } while (0)
    while (produced < count) {
        const uint32_t len = ((uint32_t)w < count - produced) ? (uint32_t)w : count - produced;
        if (pos + (uint64_t)(w / 8) > size) return fail(3, "truncated bitmask", pos);
        uint64_t bm = 0;
        for (int byte = 0; byte < w / 8; ++byte) bm |= (uint64_t)data[pos + byte] << (8 * byte);
        pos += (uint64_t)(w / 8);
        const uint64_t used = (len == 64) ? bm : (bm & ((1ULL << len) - 1));
        int set = 0;
        uint8_t info[64];
        for (uint32_t k = 0; k < len; ++k)
            if ((used >> k) & 1) {
                TAKE(info[set]);
                ++set;
            }
        int at = 0;
        for (uint32_t k = 0; k < len; ++k) {
            uint64_t diff = 1;
            if ((used >> k) & 1) {
                const uint8_t nb = info[at++];
                if (nb >= 8) {
                    diff = (uint64_t)nb - 6;
                } else {
                    diff = 0;
                    for (int p = 0; p <= nb; ++p) {
                        uint8_t v;
                        TAKE(v);
                        diff = (diff << 4) | v;
                    }
                }
            }
            running += diff;
            out[produced + k] = (uint32_t)(running - 1);
        }
        produced += len;
        if (half) ++pos, half = 0;
    }
#undef TAKE
    *consumed = pos;
    return 0;
}

/* ---------------------------------------------------------------- list build
 * neighbor_build.cpp:74-184. */
struct orc_store {
    uint64_t num_sc;
    uint32_t* counts;
    uint64_t* offsets;
    bytes_t blob;
};

typedef struct {
    uint32_t* v;
    uint64_t len, cap;
} u32vec;

static void u32push(u32vec* s, uint32_t v) {
    if (s->len == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 256;
        s->v = (uint32_t*)realloc(s->v, s->cap * 4);
    }
    s->v[s->len++] = v;
}

/* Shared body of orc_build_store (whole set) and the domain-decomposition helpers:
 * super-clusters [sc0, sc1) only; node geometry from the caller when ext_lo is
 * non-NULL; max_h_in > 0 replaces the set's max h in the periodic check; with
 * jflags non-NULL only the candidate j-clusters are flagged (halo), no store. */
static int build_impl(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                      const double* box6, const int* per, uint64_t num_nodes, const uint32_t* pbegin,
                      const uint32_t* pend, const int32_t* first_child, const double* ext_lo,
                      const double* ext_hi, const double* ext_maxh, uint32_t ci, uint32_t cj, int w,
                      int mode, int compress, double scale, uint64_t sc0, uint64_t sc1, double max_h_in,
                      uint8_t* jflags, orc_store** out) {
    /* ClusterParams (cluster.hpp:19-28), BuildParams (neighbor_store.hpp:25-28) */
    if (ci == 0 || cj == 0) return fail(1, "ClusterParams: cluster sizes must be positive", 0);
    if (64 % ci || 64 % cj) return fail(1, "ClusterParams: cluster sizes must divide the super-cluster size", 0);
    if (ci % cj) return fail(1, "ClusterParams: cj must divide ci", 0);
    if (w != 32 && w != 64) return fail(1, "ClusterParams: block width must be 32 or 64", 0);
    if (!(scale >= 1.0)) return fail(1, "BuildParams: build_radius_scale must be >= 1", 0);
    const box_t bx = mkbox(box6, per);
    const uint64_t total_sc = (n + 63) / 64;
    if (sc1 > total_sc) sc1 = total_sc;
    if (sc0 > sc1) return fail(1, "build_neighbor_store: bad super-cluster range", 0);
    const uint64_t p_lo = sc0 * 64, p_hi = sc1 * 64 < n ? sc1 * 64 : n;
    /* validate (core.hpp:201-216), over the range's own particles */
    for (uint64_t i = p_lo; i < p_hi; ++i) {
        if (!(h[i] > 0)) return fail(1, "ParticleSet: h must be positive", 0);
        const double p[3] = {x[i], y[i], z[i]};
        for (int d = 0; d < 3; ++d) {
            if (!isfinite(p[d])) return fail(1, "ParticleSet: non-finite coordinate", 0);
            if (p[d] < bx.lo[d] || p[d] > bx.hi[d]) return fail(1, "ParticleSet: position outside box (wrap first)", 0);
        }
    }
    if (num_nodes == 0 || pend[0] != (uint32_t)n) return fail(2, "build_neighbor_store: octree/particle-set mismatch", 0);
    const int symmetric = mode != 0;
    double max_h = 0;
    for (uint64_t i = p_lo; i < p_hi; ++i) max_h = dmax(max_h, h[i]);
    if (max_h_in > 0) max_h = max_h_in;
    for (int d = 0; d < 3; ++d)
        if (bx.per[d] && blen(&bx, d) < 2.0 * scale * max_h)
            return fail(2, "build_neighbor_store: periodic box must span twice the largest cutoff", 0);

    const uint64_t num_sc = sc1 - sc0, num_icl = (n + ci - 1) / ci, num_jcl = (n + cj - 1) / cj;
    const uint32_t icl_per_sc = 64 / ci, mask_bytes = (icl_per_sc + 7) / 8;
    struct orc_store* st = (struct orc_store*)calloc(1, sizeof(struct orc_store));
    st->num_sc = num_sc;
    st->counts = (uint32_t*)calloc(num_sc + 1, 4);
    st->offsets = (uint64_t*)calloc(num_sc + 1, 8);
    *out = st;
    if (n == 0 || num_sc == 0) return 0;

    /* compute_cluster_geometry (neighbor_build.cpp:19-38) */
    aabb_t* iaabb = (aabb_t*)malloc(num_icl * sizeof(aabb_t));
    aabb_t* jaabb = (aabb_t*)malloc(num_jcl * sizeof(aabb_t));
    double* imaxh = (double*)malloc(num_icl * 8);
    double* jmaxh = (double*)malloc(num_jcl * 8);
    for (uint64_t k = 0; k < num_icl; ++k) {
        iaabb[k] = aabb_empty();
        imaxh[k] = 0;
        const uint64_t e = (k + 1) * ci < n ? (k + 1) * ci : n;
        for (uint64_t i = k * ci; i < e; ++i) {
            const double p[3] = {x[i], y[i], z[i]};
            aabb_extend_pt(&iaabb[k], p);
            imaxh[k] = dmax(imaxh[k], h[i]);
        }
    }
    for (uint64_t k = 0; k < num_jcl; ++k) {
        jaabb[k] = aabb_empty();
        jmaxh[k] = 0;
        const uint64_t e = (k + 1) * cj < n ? (k + 1) * cj : n;
        for (uint64_t i = k * cj; i < e; ++i) {
            const double p[3] = {x[i], y[i], z[i]};
            aabb_extend_pt(&jaabb[k], p);
            jmaxh[k] = dmax(jmaxh[k], h[i]);
        }
    }
    /* compute_node_aabbs / compute_node_max_radius (octree.cpp:68-96) */
    aabb_t* nbox = (aabb_t*)malloc(num_nodes * sizeof(aabb_t));
    double* nmaxh = (double*)malloc(num_nodes * 8);
    for (uint64_t k = num_nodes; k-- > 0;) {
        nbox[k] = aabb_empty();
        nmaxh[k] = 0;
        if (ext_lo) {
            for (int d = 0; d < 3; ++d) nbox[k].lo[d] = ext_lo[3 * k + d], nbox[k].hi[d] = ext_hi[3 * k + d];
            nmaxh[k] = ext_maxh[k];
        } else if (first_child[k] < 0) {
            for (uint32_t i = pbegin[k]; i < pend[k]; ++i) {
                const double p[3] = {x[i], y[i], z[i]};
                aabb_extend_pt(&nbox[k], p);
                nmaxh[k] = dmax(nmaxh[k], h[i]);
            }
        } else {
            for (int c = 0; c < 8; ++c) {
                aabb_extend(&nbox[k], &nbox[first_child[k] + c]);
                nmaxh[k] = dmax(nmaxh[k], nmaxh[first_child[k] + c]);
            }
        }
    }

    u32vec cand = {0, 0, 0}, ent = {0, 0, 0};
    uint64_t* masks = NULL;
    uint64_t mask_cap = 0;
    int32_t* stack = (int32_t*)malloc((num_nodes * 8 + 16) * 4);
    for (uint64_t sc = sc0; sc < sc1; ++sc) {
        const uint64_t icl_base = sc * icl_per_sc;
        const uint64_t icl_end = icl_base + icl_per_sc < num_icl ? icl_base + icl_per_sc : num_icl;
        aabb_t sc_aabb = aabb_empty();
        double sc_maxh = 0;
        for (uint64_t gi = icl_base; gi < icl_end; ++gi) {
            aabb_extend(&sc_aabb, &iaabb[gi]);
            sc_maxh = dmax(sc_maxh, imaxh[gi]);
        }
        /* collect_candidates (neighbor_build.cpp:43-65) */
        cand.len = 0;
        uint64_t sp = 0;
        stack[sp++] = 0;
        while (sp) {
            const int32_t node = stack[--sp];
            if (pend[node] - pbegin[node] == 0) continue;
            const double r = symmetric ? scale * dmax(sc_maxh, nmaxh[node]) : scale * sc_maxh;
            if (aabb_dist_sq(&sc_aabb, &nbox[node], &bx) > r * r) continue;
            if (first_child[node] < 0) {
                const uint32_t f = pbegin[node] / cj, l = (pend[node] - 1) / cj;
                for (uint32_t j = f; j <= l; ++j)
                    if (cand.len == 0 || cand.v[cand.len - 1] != j) u32push(&cand, j);
            } else {
                for (int c = 7; c >= 0; --c) stack[sp++] = first_child[node] + c;
            }
        }
        if (jflags) {
            for (uint64_t c = 0; c < cand.len; ++c) jflags[cand.v[c]] = 1;
            continue;
        }
        /* mask loop (neighbor_build.cpp:128-161) */
        ent.len = 0;
        if (mask_cap < cand.len + 1) {
            mask_cap = cand.len + 1;
            masks = (uint64_t*)realloc(masks, mask_cap * 8);
        }
        uint64_t nmask = 0;
        for (uint64_t c = 0; c < cand.len; ++c) {
            const uint32_t jcl = cand.v[c];
            const uint64_t jb = (uint64_t)jcl * cj, je = jb + cj < n ? jb + cj : n;
            uint64_t mask = 0;
            for (uint64_t gi = icl_base; gi < icl_end; ++gi) {
                if (symmetric && gi * ci > jb) continue;
                const double pre_r = scale * (symmetric ? dmax(imaxh[gi], jmaxh[jcl]) : imaxh[gi]);
                if (aabb_dist_sq(&iaabb[gi], &jaabb[jcl], &bx) > pre_r * pre_r) continue;
                const uint64_t ib = gi * ci, ie = ib + ci < n ? ib + ci : n;
                int hit = 0;
                for (uint64_t i = ib; i < ie && !hit; ++i) {
                    const double pi_[3] = {x[i], y[i], z[i]};
                    for (uint64_t j = jb; j < je; ++j) {
                        if (i == j) continue;
                        const double r = scale * (symmetric ? dmax(h[i], h[j]) : h[i]);
                        const double pj[3] = {x[j], y[j], z[j]};
                        double d[3];
                        const double d2 = periodic_d2(pi_, pj, &bx, d);
                        if (d2 <= r * r) {
                            hit = 1;
                            break;
                        }
                    }
                }
                if (hit) mask |= 1ULL << (gi - icl_base);
            }
            if (mask) {
                u32push(&ent, jcl);
                masks[nmask++] = mask;
            }
        }
        /* serialization (neighbor_build.cpp:164-182) */
        st->counts[sc - sc0] = (uint32_t)ent.len;
        st->offsets[sc - sc0] = st->blob.len;
        for (uint64_t e = 0; e < nmask; ++e)
            for (uint32_t b = 0; b < mask_bytes; ++b) bput(&st->blob, (uint8_t)((masks[e] >> (8 * b)) & 0xff));
        if (compress) {
            const int rc = codec_encode_into(ent.v, ent.len, w, &st->blob);
            if (rc) return rc;
        } else {
            for (uint64_t e = 0; e < ent.len; ++e)
                for (int b = 0; b < 4; ++b) bput(&st->blob, (uint8_t)((ent.v[e] >> (8 * b)) & 0xff));
        }
    }
    st->offsets[num_sc] = st->blob.len;
    free(stack), free(masks), free(cand.v), free(ent.v);
    free(iaabb), free(jaabb), free(imaxh), free(jmaxh), free(nbox), free(nmaxh);
    return 0;
}

int orc_build_store(uint64_t n, const double* x, const double* y, const double* z,
                    const double* h, const double* box6, const int* per, int bits,
                    uint64_t num_nodes, const uint64_t* key_first, const uint64_t* key_last,
                    const uint32_t* pbegin, const uint32_t* pend, const int32_t* first_child,
                    uint32_t ci, uint32_t cj, int w, int mode, int compress, double scale,
                    orc_store** out) {
    (void)bits, (void)key_first, (void)key_last;
    return build_impl(n, x, y, z, h, box6, per, num_nodes, pbegin, pend, first_child, NULL, NULL, NULL, ci,
                      cj, w, mode, compress, scale, 0, (n + 63) / 64, 0.0, NULL, out);
}

int orc_build_store_range(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                          const double* box6, const int* per, uint64_t num_nodes, const uint32_t* pbegin,
                          const uint32_t* pend, const int32_t* first_child, const double* node_lo,
                          const double* node_hi, const double* node_maxh, uint32_t ci, uint32_t cj, int w,
                          int mode, int compress, double scale, uint64_t sc0, uint64_t sc1, double max_h,
                          orc_store** out) {
    return build_impl(n, x, y, z, h, box6, per, num_nodes, pbegin, pend, first_child, node_lo, node_hi,
                      node_maxh, ci, cj, w, mode, compress, scale, sc0, sc1, max_h, NULL, out);
}

int orc_halo_mark(uint64_t n, const double* x, const double* y, const double* z, const double* h,
                  const double* box6, const int* per, uint64_t num_nodes, const uint32_t* pbegin,
                  const uint32_t* pend, const int32_t* first_child, const double* node_lo,
                  const double* node_hi, const double* node_maxh, uint32_t ci, uint32_t cj, int mode,
                  double scale, uint64_t sc0, uint64_t sc1, double max_h, uint8_t* jflags) {
    orc_store* st = NULL;
    const int rc = build_impl(n, x, y, z, h, box6, per, num_nodes, pbegin, pend, first_child, node_lo, node_hi,
                              node_maxh, ci, cj, 32, mode, 1, scale, sc0, sc1, max_h, jflags, &st);
    orc_store_free(st);
    return rc;
}

void orc_store_info(const orc_store* s, uint64_t* num_sc, uint64_t* blob_size) {
    *num_sc = s->num_sc;
    *blob_size = s->blob.len;
}

void orc_store_copy(const orc_store* s, uint32_t* counts, uint64_t* offsets, uint8_t* blob) {
    memcpy(counts, s->counts, s->num_sc * 4);
    memcpy(offsets, s->offsets, (s->num_sc + 1) * 8);
    if (s->blob.len) memcpy(blob, s->blob.b, s->blob.len);
}

void orc_store_free(orc_store* s) {
    if (!s) return;
    free(s->counts), free(s->offsets), free(s->blob.b), free(s);
}

/* ---------------------------------------------------------------- pass
 * reduce.hpp:38-231 scalar path (reduce.hpp:151-197); kernels builtin_kernels.hpp:12-95.
 * neighbor_store.cpp:18-42 decode_entry_indices. */
static double min_image(double d, double len) {
    if (len > 0.0) d -= len * rint(d / len);
    return d;
}

/* sc_base: global index of the store's first super-cluster (range stores of a
 * domain decomposition, gather mode); outs/ncount are indexed from particle
 * 64 * sc_base. */
static int reduce_impl(int kernel, uint64_t n, const double* x, const double* y, const double* z,
                       const double* h, const double* m, const double* q, const double* box6,
                       const int* per, uint32_t ci, uint32_t cj, int w, int mode, int compress,
                       double scale, uint64_t sc_base, uint64_t num_sc, const uint32_t* counts,
                       const uint64_t* offsets, const uint8_t* blob, double query_scale, double eps,
                       double sigma, double ck, double** outs_g, uint32_t* ncount_g) {
    if (kernel < 0 || kernel > 3) return fail(1, "unknown kernel", 0);
    const int nout = (kernel >= 2) ? 4 : 1;
    if (query_scale > scale) return fail(1, "reduce: query_scale exceeds the store's build radius scale", 0);
    if (mode != 0 && sc_base != 0) return fail(1, "reduce: symmetric stores cannot be restricted to a range", 0);
    const uint64_t p_base = sc_base * 64;
    const uint64_t p_end = (sc_base + num_sc) * 64 < n ? (sc_base + num_sc) * 64 : n;
    const uint64_t nloc = p_end > p_base ? p_end - p_base : 0;
    for (int o = 0; o < nout; ++o) memset(outs_g[o], 0, nloc * 8);
    memset(ncount_g, 0, nloc * 4);
    if (n == 0 || nloc == 0) return 0;
    /* shift so that outs[o][i] addresses global particle i */
    double* outs[4];
    for (int o = 0; o < nout; ++o) outs[o] = outs_g[o] - p_base;
    uint32_t* ncount = ncount_g - p_base;
    counts -= sc_base;
    offsets -= sc_base;
    const box_t bx = mkbox(box6, per);
    double blen3[3];
    for (int d = 0; d < 3; ++d) blen3[d] = bx.per[d] ? blen(&bx, d) : 0.0;
    const int symmetric = mode != 0;
    const uint32_t icl_per_sc = 64 / ci, mask_bytes = (icl_per_sc + 7) / 8;
    const uint64_t num_icl = (n + ci - 1) / ci;
    const int odd[4] = {1, 1, 1, 0};
    uint32_t* idx = NULL;
    uint64_t idx_cap = 0;
    double* jacc = NULL;
    uint32_t* jcnt = NULL;
    for (uint64_t sc = sc_base; sc < sc_base + num_sc; ++sc) {
        const uint32_t count = counts[sc];
        if (!count) continue;
        if (idx_cap < count) {
            idx_cap = count;
            idx = (uint32_t*)realloc(idx, idx_cap * 4);
            jacc = (double*)realloc(jacc, idx_cap * 4 * cj * 8);
            jcnt = (uint32_t*)realloc(jcnt, idx_cap * cj * 4);
        }
        const uint64_t begin = offsets[sc], end = offsets[sc + 1];
        const uint64_t mb = (uint64_t)count * mask_bytes;
        if (begin + mb > end) return fail(3, "blob slice too short for bitmasks", begin);
        const uint8_t* rec = blob + begin;
        const uint8_t* idata = rec + mb;
        const uint64_t ilen = end - begin - mb;
        if (compress) {
            uint64_t used = 0;
            const int rc = orc_codec_decode_into(idata, ilen, count, w, idx, &used);
            if (rc) return rc;
            if (used != ilen) return fail(3, "trailing bytes in index blob", used);
        } else {
            if (ilen != (uint64_t)count * 4) return fail(3, "raw index blob length mismatch", ilen);
            memcpy(idx, idata, (size_t)count * 4);
        }
        if (symmetric) {
            memset(jacc, 0, (size_t)count * 4 * cj * 8);
            memset(jcnt, 0, (size_t)count * cj * 4);
        }
        const uint64_t icl_base = sc * icl_per_sc;
        for (uint32_t e = 0; e < count; ++e) {
            uint64_t mask = 0;
            for (uint32_t b = 0; b < mask_bytes; ++b) mask |= (uint64_t)rec[(uint64_t)e * mask_bytes + b] << (8 * b);
            const uint64_t jb = (uint64_t)idx[e] * cj, je = jb + cj < n ? jb + cj : n;
            double* acc = symmetric ? jacc + (uint64_t)e * 4 * cj : NULL;
            uint32_t* jc = symmetric ? jcnt + (uint64_t)e * cj : NULL;
            for (uint32_t b = 0; b < icl_per_sc; ++b) {
                if (!((mask >> b) & 1)) continue;
                const uint64_t gi = icl_base + b;
                if (gi >= num_icl) continue;
                const uint64_t ib = gi * ci, ie = ib + ci < n ? ib + ci : n;
                for (uint64_t i = ib; i < ie; ++i) {
                    const double hi = h[i];
                    for (uint64_t j = jb; j < je; ++j) {
                        if (i == j) continue;
                        if (symmetric && i > j && ci * (j / ci) <= cj * (i / cj)) continue;
                        const double dx = min_image(x[i] - x[j], blen3[0]);
                        const double dy = min_image(y[i] - y[j], blen3[1]);
                        const double dz = min_image(z[i] - z[j], blen3[2]);
                        const double d2 = dx * dx + dy * dy + dz * dz;
                        const double hj = h[j];
                        const double r = query_scale * (symmetric ? dmax(hi, hj) : hi);
                        if (d2 > r * r) continue;
                        double v[4] = {0, 0, 0, 0};
                        if (kernel == 0) {
                            v[0] = 1.0;
                        } else if (kernel == 1) {
                            const double rr = sqrt(d2), qq = rr / hi;
                            double wv = 0.0;
                            if (!(qq > 1.0)) {
                                const double sg = 8.0 / (kPi * hi * hi * hi);
                                if (qq <= 0.5) wv = sg * (1.0 + 6.0 * qq * qq * (qq - 1.0));
                                else {
                                    const double t = 1.0 - qq;
                                    wv = sg * 2.0 * t * t * t;
                                }
                            }
                            v[0] = m[j] * wv;
                        } else {
                            if (d2 == 0.0) return fail(1, "LjKernel: coincident particles", 0);
                            const double inv2 = 1.0 / d2;
                            const double s2 = sigma * sigma * inv2;
                            const double s6 = s2 * s2 * s2;
                            double coef = 24.0 * eps * inv2 * (2.0 * s6 * s6 - s6);
                            double en = 4.0 * eps * (s6 * s6 - s6);
                            if (kernel == 3) {
                                const double qq = ck * q[i] * q[j];
                                const double inv_r = sqrt(inv2);
                                en += qq * inv_r;
                                coef += qq * inv_r * inv2;
                            }
                            v[0] = coef * dx, v[1] = coef * dy, v[2] = coef * dz, v[3] = en;
                        }
                        for (int o = 0; o < nout; ++o) outs[o][i] = outs[o][i] + v[o];
                        ++ncount[i];
                        if (symmetric) {
                            const uint32_t lane = (uint32_t)(j - jb);
                            for (int o = 0; o < nout; ++o) {
                                const int is_odd = (kernel >= 2) && odd[o];
                                acc[o * cj + lane] = acc[o * cj + lane] + (is_odd ? -v[o] : v[o]);
                            }
                            ++jc[lane];
                        }
                    }
                }
            }
        }
        if (symmetric) { /* ordered commit (reduce.hpp:202-215) */
            for (uint32_t e = 0; e < count; ++e) {
                const uint64_t jb = (uint64_t)idx[e] * cj, je = jb + cj < n ? jb + cj : n;
                for (uint64_t j = jb; j < je; ++j) {
                    const uint32_t lane = (uint32_t)(j - jb);
                    for (int o = 0; o < nout; ++o) outs[o][j] = outs[o][j] + jacc[((uint64_t)e * 4 + o) * cj + lane];
                    ncount[j] += jcnt[(uint64_t)e * cj + lane];
                }
            }
        }
    }
    free(idx), free(jacc), free(jcnt);
    return 0;
}

int orc_reduce(int kernel, uint64_t n, const double* x, const double* y, const double* z,
               const double* h, const double* m, const double* q, const double* box6,
               const int* per, uint32_t ci, uint32_t cj, int w, int mode, int compress,
               double scale, uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
               const uint8_t* blob, uint64_t blob_size, double query_scale, double eps,
               double sigma, double ck, double** outs, uint32_t* ncount) {
    (void)blob_size;
    return reduce_impl(kernel, n, x, y, z, h, m, q, box6, per, ci, cj, w, mode, compress, scale, 0, num_sc,
                       counts, offsets, blob, query_scale, eps, sigma, ck, outs, ncount);
}

int orc_reduce_range(int kernel, uint64_t n, const double* x, const double* y, const double* z,
                     const double* h, const double* m, const double* q, const double* box6,
                     const int* per, uint32_t ci, uint32_t cj, int w, int compress, double scale,
                     uint64_t sc_base, uint64_t num_sc, const uint32_t* counts, const uint64_t* offsets,
                     const uint8_t* blob, double query_scale, double eps, double sigma, double ck,
                     double** outs, uint32_t* ncount) {
    return reduce_impl(kernel, n, x, y, z, h, m, q, box6, per, ci, cj, w, 0, compress, scale, sc_base, num_sc,
                       counts, offsets, blob, query_scale, eps, sigma, ck, outs, ncount);
}
