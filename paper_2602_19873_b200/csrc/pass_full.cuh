// Full (per-particle) Verlet list baseline: the classic LAMMPS-like list
// the paper compares the compressed clustered list against (baselines.hpp:25-131).
// Included by pass.cu (shares the store decoder and the fp64 reference kernels).
//
// build: the per-particle list of a gather store's pairs -- for every target i, every j
// of the entries carrying i's cluster bit with d2 <= (build_scale h_i)^2 (the reference
// predicate, fp64), in ascending j (entries are ascending, j ascending within a cluster):
// exactly build_full_list(ps, box, build_scale, gather) of the reference (which uses a
// cell grid; the store already holds every candidate pair). Two passes: counts ->
// exclusive scan -> fill. CSR offsets u64 [n + 1], neighbors u32.
// pass: reduce_full<Real,K> (baselines.hpp:47-129) over the CSR list -- exact query-cutoff
// filtering; precision 0: thread per i in ascending j with the reference's fp64 kernel
// expressions (bit-equal to reduce_full<double>); precision 1: warp per i (lanes stride
// the list, fp64 values, tree sum), the GPU layout a LAMMPS-like code uses. A symmetric
// full list (directed both ways, d <= scale max(h_i, h_j)) only changes the cutoff.

template <bool FILL>
__global__ void __launch_bounds__(kExactThreads) k_full_list(const __grid_constant__ PassArgs A,
                                                             uint32_t* __restrict__ counts_out,
                                                             const uint64_t* __restrict__ off,
                                                             uint32_t* __restrict__ nbrs) {
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    const uint32_t t = threadIdx.x;
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        const uint64_t i = sc * kSC + t;
        const uint32_t b = t / A.ci;
        const uint64_t gi = sc * A.icl_per_sc + b;
        const bool active = t < kSC && i < A.n && gi < A.num_icl;
        double hi = 0, xi = 0, yi = 0, zi = 0;
        if (active) hi = A.h[i], xi = A.x[i], yi = A.y[i], zi = A.z[i];
        const double r = dmul(A.qs, hi);  // qs = the store's build radius scale here
        const double r2 = dmul(r, r);
        uint32_t c = 0;
        uint64_t w = (FILL && active) ? off[i] : 0;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, &s_len);
            if (len < 0) break;
            if (!active) continue;
            for (int e = 0; e < len; ++e) {
                if (!((s_msk[e] >> b) & 1ull)) continue;
                const uint64_t jb = uint64_t(s_idx[e]) * A.cj, je = tmin<uint64_t>(jb + A.cj, A.n);
                for (uint64_t j = jb; j < je; ++j) {
                    if (i == j) continue;
                    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, nullptr, nullptr, nullptr);
                    if (d2 > r2) continue;
                    if (FILL) nbrs[w++] = uint32_t(j);
                    ++c;
                }
            }
        }
        if (!FILL && active) counts_out[i] = c;
    }
}

// reduce_full, precision 0: thread per i, ascending j, reference fp64 expressions.
template <int K>
__global__ void __launch_bounds__(128) k_reduce_full_exact(const __grid_constant__ PassArgs A, const uint64_t* __restrict__ off,
                                                           const uint32_t* __restrict__ nbrs) {
    constexpr int NO = nout<K>();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < A.n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double hi = A.h[i], xi = A.x[i], yi = A.y[i], zi = A.z[i];
        const double r = dmul(A.qs, hi), r2 = dmul(r, r);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t cnt = 0;
        bool coincident = false;
        for (uint64_t k = off[i]; k < off[i + 1]; ++k) {
            const uint64_t j = nbrs[k];
            double dx, dy, dz;
            const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
            if (A.symmetric) {
                const double rr = dmul(A.qs, smax(hi, A.h[j]));
                if (d2 > dmul(rr, rr)) continue;
            } else if (d2 > r2) continue;
            double v[4];
            if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) {
                coincident = true;
                continue;
            }
#pragma unroll
            for (int o = 0; o < NO; ++o) acc[o] = dadd(acc[o], v[o]);
            ++cnt;
        }
        if (coincident) raise_error(A.err, i / kSC, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
#pragma unroll
        for (int o = 0; o < NO; ++o) A.out[o][i] = acc[o];
        A.cnt[i] = cnt;
    }
}

// reduce_full, precision 1: warp per i, lanes stride the list, tree sum.
template <int K>
__global__ void __launch_bounds__(256) k_reduce_full_warp(const __grid_constant__ PassArgs A, const uint64_t* __restrict__ off,
                                                          const uint32_t* __restrict__ nbrs) {
    constexpr int NO = nout<K>();
    const unsigned lane = lane_id();
    const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < A.n; i += nw) {
        const double hi = A.h[i], xi = A.x[i], yi = A.y[i], zi = A.z[i];
        const double r = dmul(A.qs, hi), r2 = dmul(r, r);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t cnt = 0;
        bool coincident = false;
        for (uint64_t k = off[i] + lane; k < off[i + 1]; k += 32) {
            const uint64_t j = nbrs[k];
            double dx, dy, dz;
            const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
            if (A.symmetric) {
                const double rr = dmul(A.qs, smax(hi, A.h[j]));
                if (d2 > dmul(rr, rr)) continue;
            } else if (d2 > r2) continue;
            double v[4];
            if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) {
                coincident = true;
                continue;
            }
#pragma unroll
            for (int o = 0; o < NO; ++o) acc[o] += v[o];
            ++cnt;
        }
#pragma unroll
        for (int o = 0; o < NO; ++o)
            for (int s = 16; s > 0; s >>= 1) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], s);
        for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
        if (__any_sync(0xffffffffu, coincident) && lane == 0) raise_error(A.err, i / kSC, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        if (lane == 0) {
#pragma unroll
            for (int o = 0; o < NO; ++o) A.out[o][i] = acc[o];
            A.cnt[i] = cnt;
        }
    }
}

// cluster_overhead numerator (bench.cpp:93-122): pair slots of a gather store --
// for every entry and set mask bit b, |i-cluster b| * |j-cluster| (trailing partial
// clusters counted at their size). One CTA per SC, thread per entry of a block.
__global__ void __launch_bounds__(kExactThreads) k_cluster_slots(const __grid_constant__ PassArgs A,
                                                                 unsigned long long* __restrict__ slots) {
    __shared__ uint32_t s_idx[64];
    __shared__ unsigned long long s_msk[64];
    __shared__ int s_len;
    const uint32_t t = threadIdx.x;
    unsigned long long acc = 0;
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        for (uint32_t first = 0; first < st.count; first += uint32_t(A.w)) {
            const int len = next_block(A, sc, st, first, s_idx, s_msk, &s_len);
            if (len < 0) break;
            if (int(t) >= len) continue;
            const uint64_t jb = uint64_t(s_idx[t]) * A.cj, je = tmin<uint64_t>(jb + A.cj, A.n);
            const uint64_t cj_eff = je > jb ? je - jb : 0;
            const unsigned long long m = s_msk[t];
            for (uint32_t b = 0; b < A.icl_per_sc; ++b) {
                if (!((m >> b) & 1ull)) continue;
                const uint64_t gi = sc * A.icl_per_sc + b;
                if (gi >= A.num_icl) continue;
                const uint64_t ib = gi * A.ci, ie = tmin<uint64_t>(ib + A.ci, A.n);
                acc += (ie - ib) * cj_eff;
            }
        }
    }
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane_id() == 0 && acc) atomicAdd(slots, acc);
}
