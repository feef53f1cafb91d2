// Symmetric (half-list) pass: reduce<double> over a symmetric store,
// bit-equal to the reference's sequential ordered commit (reduce.hpp:186-218 with
// parallel_ordered, parallel.hpp:58-62: compute(sc) then commit(sc), in SC order).
// Included by pass.cu.
//
// In that order the output of particle p is ONE left fold that starts at the identity
// and takes, in sequence:
//   (a) the j-side accumulators acc[sc'][e][lane(p)] of every entry (sc', e) whose
//       j-cluster holds p, for sc' < sc(p), in (sc', e) order (commits before p's SC);
//   (b) p's own i-side pair values, in entry / j order (compute of p's SC);
//   (c) the same j-side accumulators for sc' >= sc(p) (p's own SC commits after its
//       compute, later SCs after that).
// Each accumulator is itself a fold from the identity over the entry's i particles
// (mask bits ascending, i ascending) of the signed pair values (odd outputs negated).
// The GPU restates that with three deterministic steps, no floating-point atomics:
//   1. k_sym_jside: thread per (entry, j lane) folds acc in the reference's i order and
//      records the entry's j-cluster and SC;
//   2. transpose: entries per j-cluster (count, scan, fill, per-cluster sort), so each
//      j-cluster has its entries in ascending global entry order;
//   3. k_sym_final: CTA per SC, thread per particle: (a), the i-side replay (the
//      k_pass_exact loop), (c).
// Pair values are recomputed in step 1 and step 3 with the same fp64 expressions, so
// both sides see identical values.

template <int K>
__global__ void __launch_bounds__(kExactThreads) k_sym_jside(const __grid_constant__ PassArgs A, const uint64_t* __restrict__ ebase,
                                                             double* __restrict__ jacc, uint32_t* __restrict__ jcnt,
                                                             uint32_t* __restrict__ ejcl, uint32_t* __restrict__ esc) {
    constexpr int NO = nout<K>();
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, &s_len);
            if (len < 0) break;
            for (uint32_t t = threadIdx.x; t < uint32_t(len) * A.cj; t += blockDim.x) {
                const uint32_t e = t / A.cj, lane = t % A.cj;
                const uint64_t gE = ebase[sc] + first + e;
                if (lane == 0) ejcl[gE] = s_idx[e], esc[gE] = uint32_t(sc);
                const uint64_t j = uint64_t(s_idx[e]) * A.cj + lane;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                uint32_t cnt = 0;
                if (j < A.n) {
                    const double xj = A.x[j], yj = A.y[j], zj = A.z[j], hj = A.h[j];
                    const unsigned long long m = s_msk[e];
                    for (uint32_t b = 0; b < A.icl_per_sc; ++b) {
                        if (!((m >> b) & 1ull)) continue;
                        const uint64_t gi = sc * A.icl_per_sc + b;
                        if (gi >= A.num_icl) continue;
                        const uint64_t ib = gi * A.ci, ie = tmin<uint64_t>(ib + A.ci, A.n);
                        for (uint64_t i = ib; i < ie; ++i) {
                            if (i == j) continue;
                            if (i > j && uint64_t(A.ci) * (j / A.ci) <= uint64_t(A.cj) * (i / A.cj)) continue;
                            const double hi = A.h[i];
                            double dx, dy, dz;
                            const double d2 = pair_d2_exact(A.x[i], A.y[i], A.z[i], xj, yj, zj, A.box, &dx, &dy, &dz);
                            const double rr = dmul(A.qs, smax(hi, hj));
                            if (d2 > dmul(rr, rr)) continue;
                            double v[4];
                            if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) continue;  // reported by k_sym_final
#pragma unroll
                            for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], (NO == 4 && o < 3) ? -v[o] : v[o]);
                            ++cnt;
                        }
                    }
                }
#pragma unroll
                for (int o = 0; o < NO; ++o) jacc[(gE * NO + o) * A.cj + lane] = acc[o];
                jcnt[gE * A.cj + lane] = cnt;
            }
        }
    }
}

// Entries of a super-cluster whose slice failed to decode keep ejcl = ~0 (the error is
// reported after the pass); they are left out of the lists.
__global__ void k_sym_tcount(uint64_t num_e, uint64_t ncl, const uint32_t* __restrict__ ejcl, uint32_t* __restrict__ tcnt) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < num_e; g += uint64_t(gridDim.x) * blockDim.x)
        if (ejcl[g] < ncl) atomicAdd(tcnt + ejcl[g], 1u);
}

__global__ void k_sym_tfill(uint64_t num_e, uint64_t ncl, const uint32_t* __restrict__ ejcl, const uint64_t* __restrict__ tstart,
                            uint32_t* __restrict__ tfill, uint32_t* __restrict__ tlist) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < num_e; g += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = ejcl[g];
        if (c < ncl) tlist[tstart[c] + atomicAdd(tfill + c, 1u)] = uint32_t(g);
    }
}

// per j-cluster insertion sort of its (short) entry list into ascending entry order
__global__ void k_sym_tsort(uint64_t ncl, const uint64_t* __restrict__ tstart, uint32_t* __restrict__ tlist) {
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < ncl; c += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t b = tstart[c], e = tstart[c + 1];
        for (uint64_t k = b + 1; k < e; ++k) {
            const uint32_t v = tlist[k];
            uint64_t q = k;
            while (q > b && tlist[q - 1] > v) tlist[q] = tlist[q - 1], --q;
            tlist[q] = v;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(kExactThreads) k_sym_final(const __grid_constant__ PassArgs A, const double* __restrict__ jacc,
                                                             const uint32_t* __restrict__ jcnt, const uint32_t* __restrict__ esc,
                                                             const uint64_t* __restrict__ tstart, const uint32_t* __restrict__ tlist) {
    constexpr int NO = nout<K>();
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    const uint32_t t = threadIdx.x;
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        const uint64_t i = sc * kSC + t;
        const uint32_t b = t / A.ci;
        const bool active = t < kSC && i < A.n;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t cnt = 0;
        uint64_t k = 0, kend = 0;
        const uint32_t lane = uint32_t(i % A.cj);
        auto commit = [&](bool before) {  // (a) before: entries of SCs < sc; (c) the rest
            for (; k < kend; ++k) {
                const uint32_t g = tlist[k];
                if (before && esc[g] >= sc) break;
#pragma unroll
                for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], jacc[(uint64_t(g) * NO + o) * A.cj + lane]);
                cnt += jcnt[uint64_t(g) * A.cj + lane];
            }
        };
        double hi = 0, xi = 0, yi = 0, zi = 0;
        if (active) {
            const uint64_t c = i / A.cj;
            k = tstart[c], kend = tstart[c + 1];
            commit(true);
            hi = A.h[i], xi = A.x[i], yi = A.y[i], zi = A.z[i];
        }
        bool coincident = false;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, &s_len);
            if (len < 0) break;
            if (!active) continue;
            for (int e = 0; e < len; ++e) {
                if (!((s_msk[e] >> b) & 1ull)) continue;
                const uint64_t jb = uint64_t(s_idx[e]) * A.cj, je = tmin<uint64_t>(jb + A.cj, A.n);
                for (uint64_t j = jb; j < je; ++j) {
                    if (i == j) continue;
                    if (i > j && uint64_t(A.ci) * (j / A.ci) <= uint64_t(A.cj) * (i / A.cj)) continue;
                    double dx, dy, dz;
                    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
                    const double rr = dmul(A.qs, smax(hi, A.h[j]));
                    if (d2 > dmul(rr, rr)) continue;
                    double v[4];
                    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) {
                        coincident = true;
                        continue;
                    }
#pragma unroll
                    for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], v[o]);
                    ++cnt;
                }
            }
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        if (active) {
            commit(false);
#pragma unroll
            for (int o = 0; o < NO; ++o) A.out[o][i] = acc[o];
            A.cnt[i] = cnt;
        }
    }
}
