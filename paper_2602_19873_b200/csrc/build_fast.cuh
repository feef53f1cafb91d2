// Fast interaction masks (included by build.cu inside namespace sfcnl_cu::{anon}).
//
// Gather stores with ci == 8 (cj in {4, 8}). Returns false (without touching cmask)
// for an SC that is not "safe" (below); that SC then takes the exact per-candidate
// loop of build_sc.
//
// Coordinates are made relative to the SC's first particle in fp64, min-imaged per
// particle and rounded to fp32. On periodic axes this is the true minimum image of
// every in-range pair when max|rel_i| + scale*max h < L/2 ("safe"). Then:
//  * an fp32 AABB gap between the i-cluster box and the staged j-cluster box that
//    exceeds pre_r^2 + guard proves no pair of the two clusters is within r_i, so the
//    bit is 0 whatever the reference's prefilter says (work filter only);
//  * a pair with d2_f32 < r2 - guard is within r_i in exact arithmetic, and then the
//    reference prefilter (aabb_dist_sq <= pre_r^2, pre_r >= r_i) also passes: bit 1;
//  * pairs inside the guard band are decided by the reference predicates in fp64.
// Work layout per chunk of kCh candidates: stage (thread per j slot), prefilter
// (thread per (candidate, i-cluster)), pair tests (warp per surviving pair, lane =
// 8 i x 4 j-quarters, two j slots per lane as packed f32x2, ballot any-hit).
constexpr uint32_t kCh = 64;  // candidates per staging chunk

__device__ bool fast_masks(const BuildArgs& A, const Workspace& W, uint32_t nC, uint32_t nicl,
                           uint64_t p0, uint32_t np, const double* s_x, const double* s_y,
                           const double* s_z, const double* s_h, const Geo* s_igeo) {
    // staged j slots: per (candidate, j-quarter q) 8 floats {x_a,x_b,y_a,y_b,z_a,z_b,-,-}
    // for slots a = q, b = q + 4, so each lane loads its two slots as packed pairs
    __shared__ __align__(16) float s_st[kCh * 32];
    __shared__ float s_jab[kCh][6];
    __shared__ unsigned s_pm[8][kCh / 32];  // prefilter survivors per i-cluster
    __shared__ unsigned s_self[kCh / 32];
    __shared__ unsigned s_hit[8][kCh / 32];  // pair-test hits per i-cluster
    __shared__ uint32_t s_cand[kCh];
    __shared__ float s_ix[64], s_iy[64], s_iz[64], s_lo[64], s_hi[64];
    __shared__ float s_iab[8][6];
    __shared__ float s_pthr[8];
    __shared__ float s_red[4][4];
    __shared__ int s_unsafe;
    const unsigned tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const unsigned nwarp = blockDim.x >> 5;
    const double ox = s_x[0], oy = s_y[0], oz = s_z[0];
    auto rel = [&](double v, double o, int d) {
        double r = dsub(v, o);
        if (A.box.per[d]) {
            const double L = A.box.len[d];
            if (r > 0.5 * L) r = dsub(r, L);
            else if (r < -0.5 * L) r = dadd(r, L);
        }
        return r;
    };
    float ax = 0.f, ay = 0.f, az = 0.f, ar = 0.f;
    for (uint32_t k = tid; k < 64; k += blockDim.x) {
        float fx = 1e30f, fy = 1e30f, fz = 1e30f;
        if (k < np) {
            const double qx = rel(s_x[k], ox, 0), qy = rel(s_y[k], oy, 1), qz = rel(s_z[k], oz, 2);
            fx = float(qx), fy = float(qy), fz = float(qz);
            ax = fmaxf(ax, float(fabs(qx))), ay = fmaxf(ay, float(fabs(qy))), az = fmaxf(az, float(fabs(qz)));
            ar = fmaxf(ar, float(dmul(A.scale, s_h[k])));
        }
        s_ix[k] = fx, s_iy[k] = fy, s_iz[k] = fz;
    }
    for (int o = 16; o > 0; o >>= 1) {
        ax = fmaxf(ax, __shfl_xor_sync(0xffffffffu, ax, o));
        ay = fmaxf(ay, __shfl_xor_sync(0xffffffffu, ay, o));
        az = fmaxf(az, __shfl_xor_sync(0xffffffffu, az, o));
        ar = fmaxf(ar, __shfl_xor_sync(0xffffffffu, ar, o));
    }
    if (lane == 0) s_red[warp][0] = ax, s_red[warp][1] = ay, s_red[warp][2] = az, s_red[warp][3] = ar;
    __syncthreads();
    if (tid == 0) {
        float m[4] = {0.f, 0.f, 0.f, 0.f};
        for (unsigned w = 0; w < nwarp; ++w)
            for (int k = 0; k < 4; ++k) m[k] = fmaxf(m[k], s_red[w][k]);
        int unsafe = 0;
        for (int d = 0; d < 3; ++d)
            if (A.box.per[d] && double(m[d]) + double(m[3]) >= 0.49 * A.box.len[d]) unsafe = 1;
        s_unsafe = unsafe;
        s_red[0][0] = fmaxf(m[0], fmaxf(m[1], m[2]));  // E_i
    }
    __syncthreads();
    if (s_unsafe) return false;
    const float Ei = s_red[0][0];
    if (tid < nicl) {  // fp32 boxes of the i-clusters (relative frame)
        float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
        for (uint32_t k = tid * 8; k < tmin<uint32_t>(tid * 8 + 8, np); ++k) {
            lo[0] = fminf(lo[0], s_ix[k]), hi[0] = fmaxf(hi[0], s_ix[k]);
            lo[1] = fminf(lo[1], s_iy[k]), hi[1] = fmaxf(hi[1], s_iy[k]);
            lo[2] = fminf(lo[2], s_iz[k]), hi[2] = fmaxf(hi[2], s_iz[k]);
        }
        for (int d = 0; d < 3; ++d) s_iab[tid][d] = lo[d], s_iab[tid][3 + d] = hi[d];
    }
    const uint32_t cj = A.cj;
    const uint32_t il = lane >> 2, jq = lane & 3;
    for (uint32_t c0 = 0; c0 < nC; c0 += kCh) {
        const uint32_t nc = tmin<uint32_t>(kCh, nC - c0);
        __syncthreads();  // previous chunk fully consumed
        for (uint32_t c = tid; c < nc; c += blockDim.x) s_cand[c] = W.cand[c0 + c];
        __syncthreads();
        float emax = 0.f;
        for (uint32_t t = tid; t < nc * 8; t += blockDim.x) {
            const uint32_t c = t >> 3, jj = t & 7;
            const uint32_t o = c * 32 + (jj & 3) * 8 + (jj >> 2);
            float vx = 1e30f, vy = 1e30f, vz = 1e30f;
            const uint64_t j = uint64_t(s_cand[c]) * cj + jj;
            if (jj < cj && j < A.n) {
                vx = float(rel(A.x[j], ox, 0)), vy = float(rel(A.y[j], oy, 1)), vz = float(rel(A.z[j], oz, 2));
                emax = fmaxf(emax, fmaxf(fabsf(vx), fmaxf(fabsf(vy), fabsf(vz))));
            }
            s_st[o] = vx, s_st[o + 2] = vy, s_st[o + 4] = vz;
        }
        for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        if (lane == 0) s_red[warp][1] = emax;
        __syncthreads();
        float E = Ei;
        for (unsigned w = 0; w < nwarp; ++w) E = fmaxf(E, s_red[w][1]);
        for (uint32_t c = tid; c < nc; c += blockDim.x) {  // staged j-cluster boxes
            float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
            for (uint32_t jj = 0; jj < cj; ++jj) {
                const uint32_t o = c * 32 + (jj & 3) * 8 + (jj >> 2);
                const float vx = s_st[o];
                if (vx == 1e30f) continue;
                lo[0] = fminf(lo[0], vx), hi[0] = fmaxf(hi[0], vx);
                lo[1] = fminf(lo[1], s_st[o + 2]), hi[1] = fmaxf(hi[1], s_st[o + 2]);
                lo[2] = fminf(lo[2], s_st[o + 4]), hi[2] = fmaxf(hi[2], s_st[o + 4]);
            }
            for (int d = 0; d < 3; ++d) s_jab[c][d] = lo[d], s_jab[c][3 + d] = hi[d];
        }
        if (tid < 64) {  // per-i cutoff thresholds with the guard band
            if (tid < np) {
                const double r = dmul(A.scale, s_h[tid]);
                const double r2 = dmul(r, r), g = d2_guard(r, r2, E);
                s_lo[tid] = __double2float_rd(r2 - g);
                s_hi[tid] = __double2float_ru(r2 + g);
            } else {
                s_lo[tid] = -1.f, s_hi[tid] = -1.f;
            }
        }
        if (tid < nicl) {
            const double pr = dmul(A.scale, s_igeo[tid].maxh);
            const double pr2 = dmul(pr, pr);
            s_pthr[tid] = __double2float_ru(pr2 + d2_guard(pr, pr2, E));
        }
        __syncthreads();
        // conservative fp32 prefilter -> per i-cluster bitmask over the chunk's
        // candidates (a warp covers 32 candidates of one i-cluster: one ballot)
        for (uint32_t t0 = 0; t0 < 8 * kCh; t0 += blockDim.x) {
            const uint32_t t = t0 + tid;
            const uint32_t b = t / kCh, c = t % kCh;
            bool keep = false;
            if (b < nicl && c < nc) {
                float s = 0.f;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const float g = fmaxf(fmaxf(s_iab[b][d], s_jab[c][d]) - fminf(s_iab[b][3 + d], s_jab[c][3 + d]), 0.f);
                    s = fmaf(g, g, s);
                }
                keep = !(s > s_pthr[b]);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_pm[b][c >> 5] = bal;
        }
        // self candidates: j-clusters overlapping the SC's own particles (i == j possible)
        if (tid < 2) {
            unsigned m = 0;
            for (uint32_t k = 0; k < 32; ++k) {
                const uint32_t c = tid * 32 + k;
                const int jl0 = c < nc ? int(s_cand[c]) * int(cj) - int(p0) : 1 << 20;
                if (jl0 >= -7 && jl0 < kSC) m |= 1u << k;
            }
            s_self[tid] = m;
        }
        __syncthreads();
        // warp owns i-clusters b = warp, warp + nwarp, ...: its 8 particles stay in
        // registers while it walks the candidates of its bitmask; lane = (i, j-quarter).
        // Hits collect in a register bitmask per 32 candidates (no smem atomics);
        // candidates that overlap the SC's own particles (i == j possible) take a
        // separate loop so the main loop carries no self test.
        for (uint32_t b = warp; b < nicl; b += nwarp) {
            const uint32_t li = b * 8 + il;
            const float xi = s_ix[li], yi = s_iy[li], zi = s_iz[li];
            const f2 xi2 = f2p(xi, xi), yi2 = f2p(yi, yi), zi2 = f2p(zi, zi);
            const float lo = s_lo[li], hi = s_hi[li];
            for (int half = 0; half < 2; ++half) {
                const unsigned self = s_self[half];
                unsigned todo = s_pm[b][half] & ~self;
                unsigned hits = 0;
                auto d2pair = [&](uint32_t c, float& d2a, float& d2b) {
                    const ulonglong2 P0 = reinterpret_cast<const ulonglong2*>(s_st)[c * 8 + jq * 2];
                    const f2 Pz = reinterpret_cast<const f2*>(s_st)[c * 16 + jq * 4 + 2];
                    const f2 dx = f2sub(xi2, P0.x);
                    const f2 dy = f2sub(yi2, P0.y);
                    const f2 dz = f2sub(zi2, Pz);
                    f2u(f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx))), d2a, d2b);
                };
                // guard-band pairs: the reference's fp64 predicates decide
                auto band = [&](uint32_t c, float d2a, float d2b, bool sa, bool sb) {
                    const bool band_a = !sa && !(d2a > hi), band_b = !sb && !(d2b > hi);
                    if (!__any_sync(0xffffffffu, band_a || band_b)) return false;
                    bool ex = false;
                    const uint64_t jb = uint64_t(s_cand[c]) * cj;
                    if (band_a) ex = exact_hit(A, s_x[li], s_y[li], s_z[li], s_h[li], jb + jq);
                    if (band_b && !ex) ex = exact_hit(A, s_x[li], s_y[li], s_z[li], s_h[li], jb + jq + 4);
                    if (!__any_sync(0xffffffffu, ex)) return false;
                    // the reference prefilter must pass too (neighbor_build.cpp:136-138)
                    const double pr = dmul(A.scale, s_igeo[b].maxh);
                    return !(aabb_dist_sq(s_igeo[b], A.jgeo[s_cand[c]], A.box) > dmul(pr, pr));
                };
                while (todo) {
                    const uint32_t ca = __ffs(todo) - 1;
                    todo &= todo - 1;
                    float a0, a1;
                    d2pair(half * 32 + ca, a0, a1);
                    if (todo) {  // two candidates in flight
                        const uint32_t cb = __ffs(todo) - 1;
                        todo &= todo - 1;
                        float b0, b1;
                        d2pair(half * 32 + cb, b0, b1);
                        const unsigned va = __ballot_sync(0xffffffffu, fminf(a0, a1) < lo);
                        const unsigned vb = __ballot_sync(0xffffffffu, fminf(b0, b1) < lo);
                        if (va || band(half * 32 + ca, a0, a1, false, false)) hits |= 1u << ca;
                        if (vb || band(half * 32 + cb, b0, b1, false, false)) hits |= 1u << cb;
                    } else {
                        if (__any_sync(0xffffffffu, fminf(a0, a1) < lo) || band(half * 32 + ca, a0, a1, false, false))
                            hits |= 1u << ca;
                    }
                }
                unsigned todo_self = s_pm[b][half] & self;
                while (todo_self) {
                    const uint32_t cs = __ffs(todo_self) - 1;
                    todo_self &= todo_self - 1;
                    const uint32_t c = half * 32 + cs;
                    float d2a, d2b;
                    d2pair(c, d2a, d2b);
                    const int jl0 = int(s_cand[c]) * int(cj) - int(p0);
                    const bool sa = jl0 + int(jq) == int(li), sb = jl0 + int(jq) + 4 == int(li);
                    const bool clear = (d2a < lo && !sa) || (d2b < lo && !sb);
                    if (__any_sync(0xffffffffu, clear) || band(c, d2a, d2b, sa, sb)) hits |= 1u << cs;
                }
                if (lane == 0) s_hit[b][half] = hits;
            }
        }
        __syncthreads();
        for (uint32_t c = tid; c < nc; c += blockDim.x) {
            uint32_t m = 0;
            for (uint32_t b = 0; b < nicl; ++b) m |= ((s_hit[b][c >> 5] >> (c & 31)) & 1u) << b;
            W.cmask[c0 + c] = m;
        }
    }
    __syncthreads();
    return true;
}
