// Mixed-precision neighborhood pass (precision 1), included by pass.cu inside
// namespace sfcnl_cu::{anon}. See pass.cu's header for the numerical contract.
//
// Per super-cluster (one CTA, 8 warps; warp b owns i-cluster b, lane = 8 i x 4 j-quarters):
//  1. decode: the SC's w-wide codec blocks are decoded in parallel, one warp per
//     block, using the device-side block-offset table (btab, written by the build
//     or by k_block_table for uploaded stores); SCs with more blocks than the table
//     holds fall back to a sequential decode by warp 0.
//  2. stage: every j particle of the chunk's entries is converted once to fp32
//     coordinates relative to the SC's first particle (hi part, + lo part for LJ),
//     with its payload, into shared memory.
//  3. compute: each warp walks only the entries whose mask has its bit (ballot +
//     ffs), two j slots per lane in packed f32x2 (FFMA2/FADD2/FMUL2), branch-free.
// Three block barriers per chunk of up to kCap entries (typically one chunk per SC).

constexpr int kFastThreads = 256;  // 8 warps = 8 i-clusters of 8
constexpr int kCap = 256;          // entries per chunk
constexpr int kBtab = 16;          // block offsets kept per SC
constexpr float kFar = 1.0e30f;

typedef unsigned long long f2;  // two packed fp32 lanes for the sm_100 FFMA2/FADD2/FMUL2 pipe
__device__ __forceinline__ f2 f2p(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2u(f2 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2 f2add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2fma(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float sqrt_ftz(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float fset_lt(float a, float b) {  // 1.0f if a < b else 0.0f
    float r;
    asm("set.lt.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fset_le(float a, float b) {
    float r;
    asm("set.le.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Rare slot: cutoff inside the guard band, or an LJ pair closer than 1.22 sigma
// (force-zero crossing / overflow range): the exact reference predicate and fp64
// kernel value, accumulated into the SC's shared fp64 side sums.
template <int K>
__device__ __noinline__ int rare_slot(const PassArgs& A, uint64_t i, uint64_t j, double r2,
                                      double* side) {
    if (i == j) return 0;
    const double xi = A.x[i], yi = A.y[i], zi = A.z[i], hi = A.h[i];
    double dx, dy, dz;
    const double d2 = pair_d2_exact(xi, yi, zi, A.x[j], A.y[j], A.z[j], A.box, &dx, &dy, &dz);
    if (d2 > r2) return 0;
    double v[4];
    if (eval_exact<K>(A, i, j, d2, dx, dy, dz, hi, v)) return -1;
    constexpr int NO = nout<K>();
#pragma unroll
    for (int o = 0; o < NO; ++o) atomicAdd(side + o, v[o]);
    return 1;
}

// Decode entries [c0, c0 + n) of the SC into idx/msk (smem). All warps take part.
// Returns false on a decode error (recorded). `seq` carries the sequential
// decoder's position across chunks for SCs beyond the block table.
__device__ bool decode_chunk(const PassArgs& A, uint64_t sc, const ScStream& st, uint32_t c0, uint32_t n,
                             uint32_t* idx, uint8_t* msk, uint64_t* seq_pos, uint64_t* seq_run, int* s_bad) {
    const uint32_t w = uint32_t(A.w);
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const uint32_t nwarps = blockDim.x >> 5;
    if (threadIdx.x == 0) *s_bad = 0;
    // mask records (1 byte per entry for ci = 8)
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) msk[k] = st.rec[c0 + k];
    if (!A.compress) {
        for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
            const uint8_t* p = st.idata + 4ull * (c0 + k);
            idx[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
        }
        __syncthreads();
        return true;
    }
    const uint32_t nblocks_total = (st.count + w - 1) / w;
    const uint32_t b0 = c0 / w, b1 = (c0 + n + w - 1) / w;
    __syncthreads();
    if (nblocks_total <= uint32_t(kBtab) && A.btab) {
        // parallel: warp k decodes blocks b0 + k, b0 + k + nwarps, ... each from a
        // zero running sum; block b's true values are offset by the sum of all
        // differences before it (= last value of block b-1, plus 1).
        __shared__ uint32_t s_run[kBtab];
        for (uint32_t b = b0 + warp; b < b1; b += nwarps) {
            const uint64_t pos = A.btab[sc * kBtab + b];
            const uint32_t len = tmin<uint32_t>(w, st.count - b * w);
            uint64_t off = 0;
            int msg = 0;
            uint64_t run = 0;
            const uint64_t np = warp_decode_block(st.idata, st.ilen, pos, len, int(w), run, idx + (b * w - c0), &off, &msg);
            if (np == ~0ull) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off), *s_bad = 1;
            } else if (b + 1 == nblocks_total && np != st.ilen) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, np), *s_bad = 1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t run = *seq_run;  // carried from the previous chunk of this SC
            for (uint32_t b = b0; b < b1; ++b) {
                s_run[b - b0] = uint32_t(run);
                const uint32_t last = tmin<uint32_t>(w, st.count - b * w) - 1 + b * w - c0;
                run += uint64_t(idx[last]) + 1;
            }
            *seq_run = run;
        }
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) idx[k] += s_run[(c0 + k) / w - b0];
        __syncthreads();
        return !*s_bad;
    }
    // sequential (warp 0) for SCs beyond the block table
    if (warp == 0) {
        uint64_t pos = *seq_pos, run = *seq_run;
        for (uint32_t b = b0; b < b1; ++b) {
            const uint32_t len = tmin<uint32_t>(w, st.count - b * w);
            uint64_t off = 0;
            int msg = 0;
            const uint64_t np = warp_decode_block(st.idata, st.ilen, pos, len, int(w), run, idx + (b * w - c0), &off, &msg);
            if (np == ~0ull) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off), *s_bad = 1;
                break;
            }
            pos = np;
            if (b + 1 == nblocks_total && pos != st.ilen) {
                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, pos), *s_bad = 1;
                break;
            }
        }
        if (lane == 0) *seq_pos = pos, *seq_run = run;
    }
    __syncthreads();
    return !*s_bad;
}

template <int K, int CJ>
__global__ void __launch_bounds__(kFastThreads, 3) k_pass_fast(const __grid_constant__ PassArgs A) {
    constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    constexpr int NO = nout<K>();
    extern __shared__ __align__(16) unsigned char dsm[];
    float4* s_j = reinterpret_cast<float4*>(dsm);                       // [kCap * CJ] hi + payload
    float4* s_jl = s_j + kCap * 8;                                       // [kCap * 8] lo (LJ only)
    uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_j + (LJ ? 2 : 1) * kCap * 8);  // [kCap]
    uint8_t* s_msk = reinterpret_cast<uint8_t*>(s_idx + kCap);          // [kCap]
    __shared__ double s_side[kSC][NO];
    __shared__ float s_red[8][4];
    __shared__ double s_o[3];
    __shared__ uint64_t s_seq_pos, s_seq_run;
    __shared__ int s_unsafe, s_bad;
    const unsigned tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint32_t il = lane >> 2, jq = lane & 3;
    const int i_local = int(warp * 8 + il);
    const float sig2 = float(A.sigma * A.sigma);
    const float eps24 = float(24.0 * A.eps), eps4 = float(4.0 * A.eps);
    const float close2 = 1.5f * sig2;  // (1.22 sigma)^2: LJ pairs this close go to fp64
    for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
        ScStream st;
        if (!open_sc(A, sc, st)) continue;
        const uint64_t p0 = sc * kSC;
        if (tid == 0) {
            s_o[0] = A.x[p0], s_o[1] = A.y[p0], s_o[2] = A.z[p0];
            s_seq_pos = 0, s_seq_run = 0;
        }
        for (uint32_t k = tid; k < kSC * NO; k += kFastThreads) (&s_side[0][0])[k] = 0.0;
        __syncthreads();
        const double ox = s_o[0], oy = s_o[1], oz = s_o[2];
        const uint64_t i = p0 + uint64_t(i_local);
        const bool active = i < A.n;
        auto rel = [&](double v, double o, int d) {
            double r = dsub(v, o);
            if (A.box.per[d]) {
                const double L = A.box.len[d];
                if (r > 0.5 * L) r = dsub(r, L);
                else if (r < -0.5 * L) r = dadd(r, L);
            }
            return r;
        };
        double hi = 1.0, rx = 0, ry = 0, rz = 0;
        if (active) {
            hi = A.h[i];
            rx = rel(A.x[i], ox, 0), ry = rel(A.y[i], oy, 1), rz = rel(A.z[i], oz, 2);
        }
        const double r = dmul(A.qs, hi);
        const double r2 = dmul(r, r);
        // Per-particle min-imaging against the SC origin is exact for every in-range
        // pair when max|rel_i| + max r < L/2 on each periodic axis; otherwise this SC
        // takes the exact path.
        {
            float ax = active ? float(fabs(rx)) : 0.f, ay = active ? float(fabs(ry)) : 0.f;
            float az = active ? float(fabs(rz)) : 0.f, ar = active ? float(r) : 0.f;
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
                for (int w = 0; w < 8; ++w)
                    for (int k = 0; k < 4; ++k) m[k] = fmaxf(m[k], s_red[w][k]);
                int unsafe = 0;
                for (int d = 0; d < 3; ++d)
                    if (A.box.per[d] && double(m[d]) + double(m[3]) >= 0.49 * A.box.len[d]) unsafe = 1;
                s_unsafe = unsafe;
            }
            __syncthreads();
        }
        if (s_unsafe) {
            sc_exact<K>(A, sc, st, s_idx, reinterpret_cast<unsigned long long*>(s_j), &s_bad);
            continue;
        }
        const float fxi = float(rx), fyi = float(ry), fzi = float(rz);
        const f2 xi2 = f2p(fxi, fxi), yi2 = f2p(fyi, fyi), zi2 = f2p(fzi, fzi);
        f2 lxi2 = 0, lyi2 = 0, lzi2 = 0;
        if (LJ) {
            const float lxi = float(rx - double(fxi)), lyi = float(ry - double(fyi)), lzi = float(rz - double(fzi));
            lxi2 = f2p(lxi, lxi), lyi2 = f2p(lyi, lyi), lzi2 = f2p(lzi, lzi);
        }
        const float ei = active ? fmaxf(fabsf(fxi), fmaxf(fabsf(fyi), fabsf(fzi))) : 0.f;
        const float inv_h = float(1.0 / hi);
        const f2 invh2 = f2p(inv_h, inv_h);
        f2 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;  // packed (slot a, slot b) partial sums
        uint32_t cnt = 0;
        bool coincident = false;
        for (uint32_t c0 = 0; c0 < st.count; c0 += kCap) {
            const uint32_t n = tmin<uint32_t>(kCap, st.count - c0);
            if (!decode_chunk(A, sc, st, c0, n, s_idx, s_msk, &s_seq_pos, &s_seq_run, &s_bad)) break;
            // stage every j particle of the chunk: fp64 relative -> fp32 (hi [+ lo for LJ]).
            // Layout per (entry, j-quarter q): 8 floats {x_a, x_b, y_a, y_b, z_a, z_b, m_a, m_b}
            // for slots a = q, b = q + 4, so a lane's two slots load as packed f32x2 pairs.
            float emax = 0.f;
            float* sj = reinterpret_cast<float*>(s_j);
            float* sl = reinterpret_cast<float*>(s_jl);
            for (uint32_t t = tid; t < n * 8; t += kFastThreads) {
                const uint32_t e = t >> 3, jj = t & 7;
                const uint32_t o = e * 32 + (jj & 3) * 8 + (jj >> 2);
                float vx = kFar, vy = kFar, vz = kFar, vm = 0.f, lx = 0.f, ly = 0.f, lz = 0.f;
                const uint64_t j = uint64_t(s_idx[e]) * CJ + jj;
                if (jj < uint32_t(CJ) && j < A.n) {
                    const double qx = rel(A.x[j], ox, 0), qy = rel(A.y[j], oy, 1), qz = rel(A.z[j], oz, 2);
                    vx = float(qx), vy = float(qy), vz = float(qz);
                    vm = (K == SFCNL_KERNEL_DENSITY) ? float(A.m[j]) : 0.f;
                    if (LJ) lx = float(qx - double(vx)), ly = float(qy - double(vy)), lz = float(qz - double(vz));
                    emax = fmaxf(emax, fmaxf(fabsf(vx), fmaxf(fabsf(vy), fabsf(vz))));
                }
                sj[o] = vx, sj[o + 2] = vy, sj[o + 4] = vz, sj[o + 6] = vm;
                if (LJ) sl[o] = lx, sl[o + 2] = ly, sl[o + 4] = lz;
            }
            for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            if (lane == 0) s_red[warp][0] = emax;
            __syncthreads();
            float E = ei;
#pragma unroll
            for (int k = 0; k < 8; ++k) E = fmaxf(E, s_red[k][0]);
            // rounding-error guard band for d2 (see pass.cu header)
            const double ex = 1.1920928955078125e-07 * double(E) + 5.9604644775390625e-08 * r;
            const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
            const float lo = active ? __double2float_rd(r2 - guard) : -1.f;
            const float hi_t = active ? __double2float_ru(r2 + guard) : -1.f;
            for (uint32_t g = 0; g < n; g += 32) {
                const bool mb = g + lane < n && ((s_msk[g + lane] >> warp) & 1u);
                unsigned mine = __ballot_sync(0xffffffffu, mb);
                while (mine) {
                    const uint32_t e = g + __ffs(mine) - 1;
                    mine &= mine - 1;
                    // slots a = jq, b = jq + 4 (CJ == 4: b is a far dummy), as f32x2 pairs
                    const ulonglong2 P0 = reinterpret_cast<const ulonglong2*>(s_j)[e * 8 + jq * 2];
                    const ulonglong2 P1 = reinterpret_cast<const ulonglong2*>(s_j)[e * 8 + jq * 2 + 1];
                    f2 dx = f2sub(xi2, P0.x);
                    f2 dy = f2sub(yi2, P0.y);
                    f2 dz = f2sub(zi2, P1.x);
                    if (LJ) {
                        const ulonglong2 L0 = reinterpret_cast<const ulonglong2*>(s_jl)[e * 8 + jq * 2];
                        const ulonglong2 L1 = reinterpret_cast<const ulonglong2*>(s_jl)[e * 8 + jq * 2 + 1];
                        dx = f2add(dx, f2sub(lxi2, L0.x));
                        dy = f2add(dy, f2sub(lyi2, L0.y));
                        dz = f2add(dz, f2sub(lzi2, L1.x));
                    }
                    float pma, pmb;
                    f2u(P1.y, pma, pmb);
                    const f2 d2p = f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx)));
                    float d2a, d2b;
                    f2u(d2p, d2a, d2b);
                    // i == j can only occur in the SC's own j-clusters (warp-uniform test)
                    const int jl0 = int(s_idx[e]) * CJ - int(p0);
                    bool self_a = false, self_b = false;
                    if (jl0 >= -7 && jl0 < kSC) {
                        self_a = jl0 + int(jq) == i_local;
                        self_b = CJ == 8 && jl0 + int(jq) + 4 == i_local;
                    }
                    bool in_a = d2a < lo && !self_a, in_b = d2b < lo && !self_b;
                    bool rare_a = !in_a && !(d2a > hi_t) && !self_a;
                    bool rare_b = !in_b && !(d2b > hi_t) && !self_b;
                    if (LJ) {
                        rare_a = rare_a || (in_a && d2a < close2);
                        rare_b = rare_b || (in_b && d2b < close2);
                        in_a = in_a && !(d2a < close2);
                        in_b = in_b && !(d2b < close2);
                    }
                    if (rare_a | rare_b) {
                        double* side = &s_side[i_local][0];
                        const uint64_t jb = uint64_t(s_idx[e]) * CJ;
                        if (rare_a) {
                            const int rc = rare_slot<K>(A, i, jb + jq, r2, side);
                            cnt += rc > 0, coincident |= rc < 0;
                        }
                        if (rare_b) {
                            const int rc = rare_slot<K>(A, i, jb + jq + 4, r2, side);
                            cnt += rc > 0, coincident |= rc < 0;
                        }
                    }
                    cnt += uint32_t(in_a) + uint32_t(in_b);
                    if (K == SFCNL_KERNEL_DENSITY) {
                        // W(q)/sigma_i: 1 + 6q^2(q-1) for q <= 1/2, 2(1-q)^3 otherwise
                        const f2 q = f2mul(f2p(sqrt_ftz(d2a), sqrt_ftz(d2b)), invh2);
                        const f2 q2 = f2mul(q, q);
                        const f2 wa = f2fma(f2mul(f2p(6.f, 6.f), q2), f2sub(q, f2p(1.f, 1.f)), f2p(1.f, 1.f));
                        float q0, q1;
                        f2u(q, q0, q1);
                        const f2 t = f2p(fmaxf(1.f - q0, 0.f), fmaxf(1.f - q1, 0.f));
                        const f2 wb = f2mul(f2mul(f2p(2.f, 2.f), t), f2mul(t, t));
                        float wa0, wa1, wb0, wb1;
                        f2u(wa, wa0, wa1);
                        f2u(wb, wb0, wb1);
                        const f2 w = f2p(q0 <= 0.5f ? wa0 : wb0, q1 <= 0.5f ? wa1 : wb1);
                        acc0 = f2fma(f2p(in_a ? pma : 0.f, in_b ? pmb : 0.f), w, acc0);
                    } else if (LJ) {
                        const f2 inv2 = f2p(in_a ? rcp_ftz(d2a) : 0.f, in_b ? rcp_ftz(d2b) : 0.f);  // out/rare/self -> 0
                        const f2 s2 = f2mul(f2p(sig2, sig2), inv2);
                        const f2 s6 = f2mul(f2mul(s2, s2), s2);
                        const f2 coef = f2mul(f2mul(f2mul(f2p(eps24, eps24), inv2), s6),
                                              f2fma(f2p(2.f, 2.f), s6, f2p(-1.f, -1.f)));
                        f2 ee = f2mul(f2mul(f2p(eps4, eps4), s6), f2sub(s6, f2p(1.f, 1.f)));
                        f2 cf = coef;
                        if (K == SFCNL_KERNEL_LJ_COULOMB) {
                            const uint64_t jb = uint64_t(s_idx[e]) * CJ;
                            const float qi = float(A.ck * A.q[i]);
                            const float qa = in_a ? qi * float(A.q[jb + jq]) : 0.f;
                            const float qb = (CJ == 8 && in_b) ? qi * float(A.q[jb + jq + 4]) : 0.f;
                            float ra, rb;
                            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(d2a));
                            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(d2b));
                            const f2 qr = f2mul(f2p(qa, qb), f2p(ra, rb));
                            ee = f2add(ee, qr);
                            cf = f2fma(qr, inv2, cf);
                        }
                        acc0 = f2fma(cf, dx, acc0);
                        acc1 = f2fma(cf, dy, acc1);
                        acc2 = f2fma(cf, dz, acc2);
                        acc3 = f2add(acc3, ee);
                    }
                }
            }
            __syncthreads();  // chunk buffers reused by the next chunk
        }
        if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
        // combine: slot pair, then the 4 j-quarter lanes of each i, in fp64
        double tot[4];
        const f2 accs[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            float a, b;
            f2u(accs[o], a, b);
            double v = double(a) + double(b);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            tot[o] = v;
        }
        uint32_t c = cnt;
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        if (active && jq == 0) {
            if (K == SFCNL_KERNEL_DENSITY) {
                const double sg = 8.0 / (kPi * hi * hi * hi);
                A.out[0][i] = sg * tot[0] + s_side[i_local][0];
            } else if (K == SFCNL_KERNEL_COUNT) {
                A.out[0][i] = double(c);
            } else {
#pragma unroll
                for (int o = 0; o < 4; ++o) A.out[o][i] = tot[o] + s_side[i_local][o < NO ? o : 0];
            }
            A.cnt[i] = c;
        }
        __syncthreads();  // s_side / s_o reused by the next SC
    }
}

template <int K, int CJ>
size_t fast_smem() {
    constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    return size_t(kCap) * 8 * 16 * (LJ ? 2 : 1) + size_t(kCap) * 5;
}
