// Warp-per-super-cluster list build for point clusters (ClusterParams(1, 1, w), gather),
// the paper's "no clustering" geometry (bench.cpp:227-232). Included by
// build.cu after build_warp.cuh. Same results as build_neighbor_store
// (neighbor_build.cpp:74-184) with ci = cj = 1: an SC is 64 one-particle i-clusters, every
// particle of an accepted leaf is a candidate j, and the entry mask has one bit per i.
//
//  1. SC box, traversal and candidate prefix exactly as k_build_warp (warp_bfs; with
//     cj = 1 the candidates of a leaf are its particles).
//  2. per 32 candidates (lane = candidate): the j particle relative to the SC's first
//     particle (fp64 minimum image, rounded to fp32); the 64 i rows as packed f32x2
//     pairs (two i per FFMA2) against the per-i guard-band thresholds [lo, hi] (pass.cu);
//     d2 < lo is a hit (both reference predicates hold: for points, aabb_dist_sq is the
//     squared minimum-image distance up to fp64 rounding, far inside the band), rows in
//     [lo, hi] are decided by the reference's fp64 pair predicate and prefilter.
//  3. entries (mask != 0) and their 8 mask bytes go to the warp's global workspace in
//     order, then the warp's nibble encoder writes the index list there and the record
//     is bump-allocated into the scratch (as k_build_warp).
// Unsafe SCs (ambiguous periodic images) run the reference predicates for every pair.
// SCs with more candidates than the workspace holds go to the global-memory fallback.
constexpr uint32_t kP1F = 1024;  // frontier entries per buffer (point clusters accept more leaves)

struct alignas(16) P1Smem {
    uint32_t fa[kP1F], fb[kP1F];  // traversal frontier, then per-leaf candidate prefix
    float ix[64], iy[64], iz[64], ilo[64], ihi[64];
};

__global__ void __launch_bounds__(kBwWarps * 32, 4) k_build_p1(const __grid_constant__ BuildArgs A, uint64_t sc_begin,
                                                                uint64_t sc_end, unsigned long long* __restrict__ work,
                                                                uint8_t* __restrict__ wsp, uint64_t wstride, uint32_t cap) {
    extern __shared__ __align__(16) unsigned char dsm[];
    P1Smem& S = reinterpret_cast<P1Smem*>(dsm)[threadIdx.x >> 5];
    const unsigned lane = lane_id();
    uint8_t* const base = wsp + (uint64_t(blockIdx.x) * kBwWarps + (threadIdx.x >> 5)) * wstride;
    uint32_t* const tidx = reinterpret_cast<uint32_t*>(base);                          // [cap]
    unsigned long long* const tmsk = reinterpret_cast<unsigned long long*>(base + 4ull * cap);  // [cap]
    uint8_t* const tenc = base + 12ull * cap;                                          // encoded record
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(work, 1ull);
        const uint64_t sc = sc_begin + __shfl_sync(0xffffffffu, t, 0);
        if (sc >= sc_end) break;
        bool ok = true;
        const uint64_t icl_base = sc * 64;
        const uint32_t nicl = uint32_t(tmin<uint64_t>(icl_base + 64, A.num_icl) - icl_base);
        const uint64_t p0 = icl_base;
        // ---- 1. SC box and i side
        Geo scg;
        double r2;
        sc_box(A, icl_base, nicl, scg, r2);
        const double ox = A.x[p0], oy = A.y[p0], oz = A.z[p0];
        auto rel = [&](double v, double o, int d) {
            double r = dsub(v, o);
            if (A.box.per[d]) {
                const double L = A.box.len[d];
                if (r > 0.5 * L) r = dsub(r, L);
                else if (r < -0.5 * L) r = dadd(r, L);
            }
            return r;
        };
        float eax = 0.f, eay = 0.f, eaz = 0.f, er = 0.f;
        double ri[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const uint32_t k = lane + 32u * s;
            float fx = 1e30f, fy = 1e30f, fz = 1e30f;
            ri[s] = -1.0;
            if (k < nicl) {
                const double qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                fx = float(qx), fy = float(qy), fz = float(qz);
                eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                ri[s] = dmul(A.scale, A.h[p0 + k]);
                er = fmaxf(er, float(ri[s]));
            }
            S.ix[k] = fx, S.iy[k] = fy, S.iz[k] = fz;
        }
        eax = warp_fmax(eax), eay = warp_fmax(eay), eaz = warp_fmax(eaz), er = warp_fmax(er);
        const bool unsafe = (A.box.per[0] && double(eax) + double(er) >= 0.49 * A.box.len[0]) ||
                            (A.box.per[1] && double(eay) + double(er) >= 0.49 * A.box.len[1]) ||
                            (A.box.per[2] && double(eaz) + double(er) >= 0.49 * A.box.len[2]);
        const float Ei = fmaxf(eax, fmaxf(eay, eaz));
        __syncwarp();
        // ---- traversal and candidate prefix (as build_sc_warp, cj = 1)
        uint32_t* fa;
        const uint32_t nA = warp_bfs(A, scg, r2, S.fa, S.fb, &fa, kP1F);
        uint32_t nC = 0;
        uint32_t* fb = nullptr;
        if (nA == ~0u) {
            ok = false;
        } else {
            fb = fa == S.fa ? S.fb : S.fa;
            uint32_t prev_last = 0xffffffffu;
            for (uint32_t b0 = 0; b0 < nA; b0 += 32) {
                const uint32_t k = b0 + lane;
                uint32_t f = 0, l = 0;
                if (k < nA) {
                    const Node nd = A.nodes[fa[k] & ~kTag];
                    f = nd.pbegin, l = nd.pend - 1;
                }
                uint32_t pl = __shfl_up_sync(0xffffffffu, l, 1);
                if (lane == 0) pl = prev_last;
                uint32_t start = f, cnt = 0;
                if (k < nA) {
                    if (k > 0 && pl == f) start = f + 1;
                    cnt = l + 1 - start;
                }
                const uint32_t inc = warp_incl_scan(cnt);
                __syncwarp();
                if (k < nA) fa[k] = start, fb[k] = nC + inc - cnt;
                nC += __shfl_sync(0xffffffffu, inc, 31);
                prev_last = __shfl_sync(0xffffffffu, l, 31);
            }
            __syncwarp();
            if (nC > cap) ok = false;
        }
        // ---- 2. masks, 32 candidates at a time
        uint32_t nE = 0;
        float Ej_run = -1.f;
        for (uint32_t c0 = 0; ok && c0 < nC; c0 += 32) {
            const uint32_t n = tmin<uint32_t>(32, nC - c0);
            const bool valid = lane < n;
            uint32_t cand = 0;
            if (valid) {
                const uint32_t pos = c0 + lane;
                uint32_t lo = 0, hi = nA;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (fb[mid] <= pos) lo = mid;
                    else hi = mid;
                }
                cand = fa[lo] + (pos - fb[lo]);
            }
            const uint64_t j = cand;
            unsigned long long mask = 0, band = 0;
            if (unsafe) {
                if (valid) {
                    const Geo jg = A.jgeo[j];
                    for (uint32_t b = 0; b < nicl; ++b) {
                        const uint64_t i = p0 + b;
                        if (i == j) continue;
                        const Geo ig = A.igeo[icl_base + b];
                        const double pre_r = dmul(A.scale, ig.maxh);
                        if (aabb_dist_sq(ig, jg, A.box) > dmul(pre_r, pre_r)) continue;
                        const double rr = dmul(A.scale, A.h[i]);
                        const double d2 = pair_d2_exact(A.x[i], A.y[i], A.z[i], A.x[j], A.y[j], A.z[j], A.box, nullptr, nullptr, nullptr);
                        if (d2 <= dmul(rr, rr)) mask |= 1ull << b;
                    }
                }
            } else {
                float sx = 1e30f, sy = 1e30f, sz = 1e30f;
                if (valid) sx = float(rel(A.x[j], ox, 0)), sy = float(rel(A.y[j], oy, 1)), sz = float(rel(A.z[j], oz, 2));
                const float Ej = warp_fmax(valid ? fmaxf(fabsf(sx), fmaxf(fabsf(sy), fabsf(sz))) : 0.f);
                if (Ej > Ej_run) {  // thresholds for a running bound of the staged |coordinates|
                    __syncwarp();      // every lane is done with the previous chunk's thresholds
                    Ej_run = fmaxf(Ej, Ej_run * 1.0625f);
                    const double ecoord = 5.9604644775390625e-08 * (double(Ei) + double(Ej_run));
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const uint32_t k = lane + 32u * s;
                        float lo = -1.f, hi = -1.f;
                        if (ri[s] >= 0.0) {
                            const double rr2 = dmul(ri[s], ri[s]), g = guard_band(ri[s], rr2, ecoord);
                            lo = __double2float_rd(rr2 - g);
                            hi = __double2float_ru(rr2 + g);
                        }
                        S.ilo[k] = lo, S.ihi[k] = hi;
                    }
                }
                __syncwarp();
                const f2 x2 = f2p(sx, sx), y2 = f2p(sy, sy), z2 = f2p(sz, sz);
                const int self = int(int64_t(j) - int64_t(p0));  // i == j row (if inside the SC)
#pragma unroll 4
                for (uint32_t b = 0; b < 64; b += 2) {
                    const f2 xi = *reinterpret_cast<const f2*>(&S.ix[b]), yi = *reinterpret_cast<const f2*>(&S.iy[b]);
                    const f2 zi = *reinterpret_cast<const f2*>(&S.iz[b]);
                    const f2 dx = f2sub(xi, x2), dy = f2sub(yi, y2), dz = f2sub(zi, z2);
                    float d2a, d2b;
                    f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                    if (self == int(b)) d2a = 3.0e38f;
                    if (self == int(b) + 1) d2b = 3.0e38f;
                    const float2 lo = *reinterpret_cast<const float2*>(&S.ilo[b]), hi = *reinterpret_cast<const float2*>(&S.ihi[b]);
                    const unsigned long long ha = d2a < lo.x, hb = d2b < lo.y;
                    const unsigned long long ba = !(d2a < lo.x) & (d2a <= hi.x), bbn = !(d2b < lo.y) & (d2b <= hi.y);
                    mask |= (ha << b) | (hb << (b + 1));
                    band |= (ba << b) | (bbn << (b + 1));
                }
                if (!valid) mask = 0, band = 0;
                if (band) {  // guard band: the reference's pair predicate and prefilter
                    const Geo jg = A.jgeo[j];
                    for (unsigned long long m = band; m; m &= m - 1) {
                        const uint32_t b = __ffsll(m) - 1;
                        const uint64_t i = p0 + b;
                        const double rr = dmul(A.scale, A.h[i]);
                        const double d2 = pair_d2_exact(A.x[i], A.y[i], A.z[i], A.x[j], A.y[j], A.z[j], A.box, nullptr, nullptr, nullptr);
                        if (!(d2 <= dmul(rr, rr))) continue;
                        const Geo ig = A.igeo[icl_base + b];
                        const double pr = dmul(A.scale, ig.maxh);
                        if (!(aabb_dist_sq(ig, jg, A.box) > dmul(pr, pr))) mask |= 1ull << b;
                    }
                }
            }
            // ordered compaction into the workspace
            const bool keep = valid && mask != 0;
            const unsigned kb = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t at = nE + __popc(kb & lanemask_lt());
                tidx[at] = A.lc2g ? A.lc2g[cand] : cand, tmsk[at] = mask;
            }
            nE += __popc(kb);
        }
        __syncwarp();
        // ---- 3. serialization: 8 mask bytes per entry, then the index list
        uint32_t size = 0;
        if (ok) {
            const uint32_t mbytes = 8 * nE;
            for (uint32_t k = lane; k < nE; k += 32) reinterpret_cast<unsigned long long*>(tenc)[k] = tmsk[k];
            uint32_t pos = mbytes;
            if (!A.compress) {
                for (uint32_t k = lane; k < nE; k += 32) reinterpret_cast<uint32_t*>(tenc + mbytes)[k] = tidx[k];
                pos = mbytes + 4 * nE;
            } else {
                const uint32_t w = uint32_t(A.w);
                for (uint32_t bb = 0; bb < nE; bb += w) {
                    const uint32_t len = min(w, nE - bb);
                    uint64_t dv[2];
                    uint32_t nd[2], isset[2];
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const uint32_t k = lane + 32u * s;
                        dv[s] = 1, nd[s] = 0, isset[s] = 0;
                        if (k < len && (s == 0 || w == 64)) {
                            const uint64_t cur = tidx[bb + k];
                            dv[s] = (bb + k == 0) ? cur + 1 : cur - uint64_t(tidx[bb + k - 1]);
                            isset[s] = dv[s] != 1;
                            nd[s] = (dv[s] > 9) ? uint32_t(nibble_count(dv[s])) : 0u;
                        }
                    }
                    const unsigned m0 = __ballot_sync(0xffffffffu, isset[0]);
                    const unsigned m1 = __ballot_sync(0xffffffffu, isset[1]);
                    const uint32_t ninfo = __popc(m0) + __popc(m1);
                    const uint32_t inc0 = warp_incl_scan(nd[0]);
                    const uint32_t tot0 = __shfl_sync(0xffffffffu, inc0, 31);
                    const uint32_t inc1 = warp_incl_scan(nd[1]);
                    const uint32_t nib = ninfo + tot0 + __shfl_sync(0xffffffffu, inc1, 31);
                    const uint32_t bsize = w / 8 + (nib + 1) / 2;
                    const unsigned long long bm = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
                    if (lane < w / 8) tenc[pos + lane] = uint8_t(bm >> (8 * lane));
                    for (uint32_t q = lane; q < (nib + 1) / 2 + 4; q += 32) tenc[pos + w / 8 + q] = 0;
                    __syncwarp();
                    const uint32_t nbase = (pos + w / 8) * 2;
                    unsigned int* words = reinterpret_cast<unsigned int*>(tenc);
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        if (!isset[s]) continue;
                        const uint32_t info_at = s == 0 ? __popc(m0 & lanemask_lt()) : __popc(m0) + __popc(m1 & lanemask_lt());
                        const uint64_t v = dv[s];
                        const uint32_t infov = v <= 9 ? uint32_t(v + 6) : nd[s] - 1;
                        uint32_t t2 = nbase + info_at;
                        atomicOr(&words[t2 >> 3], infov << (4 * (t2 & 7)));
                        if (nd[s]) {
                            uint32_t dstart = ninfo + (s == 0 ? inc0 - nd[0] : tot0 + inc1 - nd[1]);
                            for (int p = int(nd[s]) - 1; p >= 0; --p, ++dstart) {
                                t2 = nbase + dstart;
                                atomicOr(&words[t2 >> 3], uint32_t((v >> (4 * p)) & 15u) << (4 * (t2 & 7)));
                            }
                        }
                    }
                    __syncwarp();
                    pos += bsize;
                }
            }
            size = pos;
        }
        // ---- publish (bump-allocate the scratch and copy), or hand the SC to the fallback
        unsigned long long off = 0;
        if (lane == 0) {
            if (!ok) {
                const unsigned long long slot = atomicAdd(&A.ctl[1], 1ull);
                A.overflow_list[slot] = uint32_t(sc);
                A.counts[sc] = 0, A.sizes[sc] = 0, A.soff[sc] = 0;
                off = ~0ull;
            } else {
                const unsigned long long need = (size + 15ull) & ~15ull;
                off = atomicAdd(&A.ctl[0], need);
                if (off + need > A.scratch_cap) {
                    A.ctl[2] = 1;
                    off = ~0ull;
                }
                A.counts[sc] = nE;
                A.sizes[sc] = size;
                A.soff[sc] = off;
            }
        }
        off = __shfl_sync(0xffffffffu, off, 0);
        if (ok && off != ~0ull) {
            const unsigned int* src = reinterpret_cast<const unsigned int*>(tenc);
            unsigned int* dst = reinterpret_cast<unsigned int*>(A.scratch + off);
            for (uint32_t q = lane; q < (size + 3) / 4; q += 32) dst[q] = src[q];
        }
        __syncwarp();
    }
}
