// Warp-specialized mixed-precision pass (precision 1), included by pass.cu after
// pass_fast.cuh (shares its helpers).
//
// CTA = 8 consumer warps (warp b owns i-cluster b; lane = 8 i x 4 j-quarters) +
// 2 producer warps. Producers walk the CTA's super-clusters chunk by chunk
// (<= kCap entries): decode the codec blocks in parallel from the device block
// table, stage every j particle as SC-relative fp32 (hi [+ lo for LJ]) in the
// packed-pair layout, stage the SC's own particles, and hand the chunk over through
// a double buffer. Consumers run the barrier-free per-warp pair loop of
// k_pass_fast on the buffer while producers fill the other one. Hand-over uses
// named barriers: FULL[b] (producers arrive, consumers sync) and EMPTY[b]
// (consumers arrive, producers sync), 320 threads each.
//
// Unsafe SCs (periodic images ambiguous in the SC-relative frame) are not staged
// for the fast path: the producer flags them and every slot of such an SC goes
// through the exact fp64 reference predicate + kernel (rare_slot).

constexpr int kWsConsumers = 256, kWsProducers = 128, kWsThreads = kWsConsumers + kWsProducers;
constexpr int kWsCap = 128;  // entries per chunk (double-buffered)


__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct WsMeta {
    uint64_t sc;
    uint32_t n, c0;
    int first, last, unsafe, bad;
    float E;
    double o[3];
};

template <int K>
struct WsStage {
    static constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    float sj[kWsCap * 32];
    float sl[LJ ? kWsCap * 32 : 4];
    uint32_t idx[kWsCap];
    uint8_t msk[kWsCap];
    // the SC's own particles (valid when meta.first)
    float ix[64], iy[64], iz[64], ilx[64], ily[64], ilz[64];
    double ih[64];
};

template <int K, int CJ>
__global__ void __launch_bounds__(kWsThreads, 2) k_pass_ws(const __grid_constant__ PassArgs A) {
    constexpr bool LJ = (K == SFCNL_KERNEL_LJ || K == SFCNL_KERNEL_LJ_COULOMB);
    constexpr int NO = nout<K>();
    extern __shared__ __align__(16) unsigned char dsm[];
    WsStage<K>* stg = reinterpret_cast<WsStage<K>*>(dsm);  // [2]
    __shared__ WsMeta meta[2];
    __shared__ double s_side[kSC][NO];
    __shared__ uint32_t s_run[kBtab];
    __shared__ float s_pred[kWsProducers / 32][4];
    __shared__ uint64_t s_seq_pos, s_seq_run;
    __shared__ int s_bad, s_unsafe_p;
    __shared__ float s_ei_p, s_ax[kWsProducers / 32][3];
    const unsigned tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint32_t w = uint32_t(A.w);

    if (warp >= 8) {
        // ============================ producers ============================
        const unsigned ptid = tid - kWsConsumers, pwarp = warp - 8;
        int buf = 0;
        int uses[2] = {0, 0};
        for (uint64_t sc = A.sc_begin + blockIdx.x; sc < A.num_sc; sc += gridDim.x) {
            ScStream st;
            const bool ok = open_sc(A, sc, st);
            const uint32_t nchunks = (ok && st.count) ? (st.count + kWsCap - 1) / kWsCap : 1;
            const uint64_t p0 = sc * kSC;
            const uint32_t np = uint32_t(tmin<uint64_t>(p0 + kSC, A.n) - p0);
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
            if (ptid == 0) s_seq_pos = 0, s_seq_run = 0;
            for (uint32_t ch = 0; ch < nchunks; ++ch) {
                if (uses[buf]) nbar_sync(3 + buf, kWsThreads);  // EMPTY[buf]
                ++uses[buf];
                WsStage<K>& S = stg[buf];
                const uint32_t c0 = ch * kWsCap;
                const uint32_t n = (ok && st.count) ? tmin<uint32_t>(kWsCap, st.count - c0) : 0;
                float ei = 0.f, er = 0.f, eax = 0.f, eay = 0.f, eaz = 0.f;
                if (ch == 0) {  // the SC's own particles
                    for (uint32_t k = ptid; k < 64; k += kWsProducers) {
                        float fx = 0.f, fy = 0.f, fz = 0.f, lx = 0.f, ly = 0.f, lz = 0.f;
                        double hk = 1.0;
                        if (k < np) {
                            const double qx = rel(A.x[p0 + k], ox, 0), qy = rel(A.y[p0 + k], oy, 1), qz = rel(A.z[p0 + k], oz, 2);
                            fx = float(qx), fy = float(qy), fz = float(qz);
                            lx = float(qx - double(fx)), ly = float(qy - double(fy)), lz = float(qz - double(fz));
                            hk = A.h[p0 + k];
                            eax = fmaxf(eax, float(fabs(qx))), eay = fmaxf(eay, float(fabs(qy))), eaz = fmaxf(eaz, float(fabs(qz)));
                            er = fmaxf(er, float(dmul(A.qs, hk)));
                        }
                        S.ix[k] = fx, S.iy[k] = fy, S.iz[k] = fz, S.ilx[k] = lx, S.ily[k] = ly, S.ilz[k] = lz, S.ih[k] = hk;
                    }
                    ei = fmaxf(eax, fmaxf(eay, eaz));
                }
                // decode the chunk (both producer warps)
                if (ptid == 0) s_bad = 0;
                for (uint32_t k = ptid; k < n; k += kWsProducers) S.msk[k] = st.rec[c0 + k];
                nbar_sync(7, kWsProducers);
                if (n && !A.compress) {
                    for (uint32_t k = ptid; k < n; k += kWsProducers) {
                        const uint8_t* p = st.idata + 4ull * (c0 + k);
                        S.idx[k] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
                    }
                } else if (n) {
                    const uint32_t nbt = (st.count + w - 1) / w;
                    const uint32_t b0 = c0 / w, b1 = (c0 + n + w - 1) / w;
                    if (nbt <= uint32_t(kBtab) && A.btab) {
                        for (uint32_t b = b0 + pwarp; b < b1; b += kWsProducers / 32) {
                            uint64_t off = 0, run = 0;
                            int msg = 0;
                            const uint64_t np2 = warp_decode_block(st.idata, st.ilen, A.btab[sc * kBtab + b],
                                                                   tmin<uint32_t>(w, st.count - b * w), int(w), run,
                                                                   S.idx + (b * w - c0), &off, &msg);
                            if (np2 == ~0ull) {
                                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off), s_bad = 1;
                            } else if (b + 1 == nbt && np2 != st.ilen) {
                                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, np2), s_bad = 1;
                            }
                        }
                        nbar_sync(7, kWsProducers);
                        if (ptid == 0) {
                            uint64_t run = s_seq_run;
                            for (uint32_t b = b0; b < b1; ++b) {
                                s_run[b - b0] = uint32_t(run);
                                run += uint64_t(S.idx[tmin<uint32_t>(w, st.count - b * w) - 1 + b * w - c0]) + 1;
                            }
                            s_seq_run = run;
                        }
                        nbar_sync(7, kWsProducers);
                        for (uint32_t k = ptid; k < n; k += kWsProducers) S.idx[k] += s_run[(c0 + k) / w - b0];
                    } else if (pwarp == 0) {
                        uint64_t pos = s_seq_pos, run = s_seq_run;
                        for (uint32_t b = b0; b < b1; ++b) {
                            uint64_t off = 0;
                            int msg = 0;
                            const uint64_t np2 = warp_decode_block(st.idata, st.ilen, pos, tmin<uint32_t>(w, st.count - b * w),
                                                                   int(w), run, S.idx + (b * w - c0), &off, &msg);
                            if (np2 == ~0ull) {
                                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, msg, off), s_bad = 1;
                                break;
                            }
                            pos = np2;
                            if (b + 1 == nbt && pos != st.ilen) {
                                if (lane == 0) raise_error(A.err, sc, SFCNL_DECODE_ERROR, kMsgTrailing, pos), s_bad = 1;
                                break;
                            }
                        }
                        if (lane == 0) s_seq_pos = pos, s_seq_run = run;
                    }
                }
                nbar_sync(7, kWsProducers);
                // stage the chunk's j particles (packed-pair layout, see k_pass_fast)
                float emax = 0.f;
                if (!s_bad) {
                    for (uint32_t t = ptid; t < n * 8; t += kWsProducers) {
                        const uint32_t e = t >> 3, jj = t & 7;
                        const uint32_t o = e * 32 + (jj & 3) * 8 + (jj >> 2);
                        float vx = kFar, vy = kFar, vz = kFar, vm = 0.f, lx = 0.f, ly = 0.f, lz = 0.f;
                        const uint64_t j = uint64_t(S.idx[e]) * CJ + jj;
                        if (jj < uint32_t(CJ) && j < A.n) {
                            const double qx = rel(A.x[j], ox, 0), qy = rel(A.y[j], oy, 1), qz = rel(A.z[j], oz, 2);
                            vx = float(qx), vy = float(qy), vz = float(qz);
                            vm = (K == SFCNL_KERNEL_DENSITY) ? float(A.m[j]) : 0.f;
                            if (LJ) lx = float(qx - double(vx)), ly = float(qy - double(vy)), lz = float(qz - double(vz));
                            emax = fmaxf(emax, fmaxf(fabsf(vx), fmaxf(fabsf(vy), fabsf(vz))));
                        }
                        S.sj[o] = vx, S.sj[o + 2] = vy, S.sj[o + 4] = vz, S.sj[o + 6] = vm;
                        if (LJ) S.sl[o] = lx, S.sl[o + 2] = ly, S.sl[o + 4] = lz;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
                    ei = fmaxf(ei, __shfl_xor_sync(0xffffffffu, ei, o));
                    er = fmaxf(er, __shfl_xor_sync(0xffffffffu, er, o));
                    eax = fmaxf(eax, __shfl_xor_sync(0xffffffffu, eax, o));
                    eay = fmaxf(eay, __shfl_xor_sync(0xffffffffu, eay, o));
                    eaz = fmaxf(eaz, __shfl_xor_sync(0xffffffffu, eaz, o));
                }
                if (lane == 0) {
                    s_pred[pwarp][0] = emax, s_pred[pwarp][1] = ei, s_pred[pwarp][2] = er;
                    s_pred[pwarp][3] = fmaxf(eax, fmaxf(eay, eaz));
                }
                if (lane == 0) s_ax[pwarp][0] = eax, s_ax[pwarp][1] = eay, s_ax[pwarp][2] = eaz;
                nbar_sync(7, kWsProducers);
                if (ptid == 0) {
                    WsMeta& M = meta[buf];
                    M.sc = sc, M.n = n, M.c0 = c0;
                    M.first = ch == 0, M.last = ch + 1 == nchunks;
                    M.bad = !ok || s_bad;
                    M.o[0] = ox, M.o[1] = oy, M.o[2] = oz;
                    if (ch == 0) {  // SC-wide: E_i and the periodic-image safety test
                        float er2 = 0.f, eim = 0.f, axm[3] = {0.f, 0.f, 0.f};
                        for (int q = 0; q < kWsProducers / 32; ++q) {
                            er2 = fmaxf(er2, s_pred[q][2]), eim = fmaxf(eim, s_pred[q][1]);
                            for (int d = 0; d < 3; ++d) axm[d] = fmaxf(axm[d], s_ax[q][d]);
                        }
                        int unsafe = 0;
                        for (int d = 0; d < 3; ++d)
                            if (A.box.per[d] &&
                                double(axm[d]) + double(er2) >= 0.49 * A.box.len[d])
                                unsafe = 1;
                        s_ei_p = eim;
                        s_unsafe_p = unsafe;
                    }
                    M.unsafe = s_unsafe_p;
                    float em = 0.f;
                    for (int q = 0; q < kWsProducers / 32; ++q) em = fmaxf(em, s_pred[q][0]);
                    M.E = fmaxf(s_ei_p, em);
                }
                nbar_arrive(1 + buf, kWsThreads);  // FULL[buf]
                buf ^= 1;
            }
        }
        // consume the consumers' final EMPTY arrivals
        for (int b = 0; b < 2; ++b)
            if (uses[b]) nbar_sync(3 + b, kWsThreads);
        return;
    }

    // ============================ consumers ============================
    const uint32_t il = lane >> 2, jq = lane & 3;
    const int i_local = int(warp * 8 + il);
    const float sig2 = float(A.sigma * A.sigma);
    const float eps24 = float(24.0 * A.eps), eps4 = float(4.0 * A.eps);
    const float close2 = 1.5f * sig2;
    int buf = 0;
    f2 xi2 = 0, yi2 = 0, zi2 = 0, lxi2 = 0, lyi2 = 0, lzi2 = 0;
    double hi = 1.0, r = 0.0, r2 = 0.0;
    f2 invh2 = 0;
    bool active = false, unsafe = false;
    uint64_t i = 0, p0 = 0;
    f2 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    uint32_t cnt = 0;
    bool coincident = false, bad = false;
    for (;;) {
        nbar_sync(1 + buf, kWsThreads);  // FULL[buf]
        const WsMeta& M = meta[buf];
        WsStage<K>& S = stg[buf];
        if (M.first) {
            p0 = M.sc * kSC;
            i = p0 + uint64_t(i_local);
            active = i < A.n;
            unsafe = M.unsafe;
            bad = false;
            hi = S.ih[i_local];
            r = dmul(A.qs, hi);
            r2 = dmul(r, r);
            const float fxi = S.ix[i_local], fyi = S.iy[i_local], fzi = S.iz[i_local];
            xi2 = f2p(fxi, fxi), yi2 = f2p(fyi, fyi), zi2 = f2p(fzi, fzi);
            if (LJ) {
                lxi2 = f2p(S.ilx[i_local], S.ilx[i_local]);
                lyi2 = f2p(S.ily[i_local], S.ily[i_local]);
                lzi2 = f2p(S.ilz[i_local], S.ilz[i_local]);
            }
            const float inv_h = float(1.0 / hi);
            invh2 = f2p(inv_h, inv_h);
            acc0 = acc1 = acc2 = acc3 = 0;
            cnt = 0;
            coincident = false;
            // s_side rows of this warp's i-cluster are private to the warp
            for (uint32_t k = lane; k < 8 * NO; k += 32) (&s_side[warp * 8][0])[k] = 0.0;
            __syncwarp();
        }
        bad |= bool(M.bad);
        const uint32_t n = M.n;
        float lo = -1.f, hi_t = -1.f;
        if (active && !bad) {
            if (!unsafe) {
                const double ex = 1.1920928955078125e-07 * double(M.E) + 5.9604644775390625e-08 * r;
                const double guard = 4.0 * (1.7881393432617188e-07 * r2 + 3.5 * r * ex + 3.0 * ex * ex) + 1e-300;
                lo = __double2float_rd(r2 - guard);
                hi_t = __double2float_ru(r2 + guard);
            }
        }
        if (!bad) {
            // one entry = 8 i x 8 j slots of this warp's i-cluster; lane (i, jq) owns
            // slots a = jq, b = jq + 4 as packed f32x2
            struct Ld {
                f2 dx, dy, dz;
                float pma, pmb, d2a, d2b;
            };
            auto load = [&](uint32_t e) {
                Ld L;
                const ulonglong2 P0 = reinterpret_cast<const ulonglong2*>(S.sj)[e * 8 + jq * 2];
                const ulonglong2 P1 = reinterpret_cast<const ulonglong2*>(S.sj)[e * 8 + jq * 2 + 1];
                L.dx = f2sub(xi2, P0.x);
                L.dy = f2sub(yi2, P0.y);
                L.dz = f2sub(zi2, P1.x);
                if (LJ) {
                    const ulonglong2 L0 = reinterpret_cast<const ulonglong2*>(S.sl)[e * 8 + jq * 2];
                    const ulonglong2 L1 = reinterpret_cast<const ulonglong2*>(S.sl)[e * 8 + jq * 2 + 1];
                    L.dx = f2add(L.dx, f2sub(lxi2, L0.x));
                    L.dy = f2add(L.dy, f2sub(lyi2, L0.y));
                    L.dz = f2add(L.dz, f2sub(lzi2, L1.x));
                }
                f2u(P1.y, L.pma, L.pmb);
                f2u(f2fma(L.dz, L.dz, f2fma(L.dy, L.dy, f2mul(L.dx, L.dx))), L.d2a, L.d2b);
                return L;
            };
            // kSelf: the entry's j-cluster overlaps the SC's own particles (i == j
            // possible); kUnsafe: periodic images ambiguous, every slot exact
            auto compute = [&](uint32_t e, const Ld& L, auto SELF, auto UNSAFE) {
                constexpr bool kSelf = decltype(SELF)::value, kUnsafe = decltype(UNSAFE)::value;
                bool self_a = false, self_b = false;
                if (kSelf) {
                    const int jl0 = int(S.idx[e]) * CJ - int(p0);
                    self_a = jl0 + int(jq) == i_local;
                    self_b = CJ == 8 && jl0 + int(jq) + 4 == i_local;
                }
                bool in_a, in_b, rare_a, rare_b;
                if (kUnsafe) {
                    in_a = in_b = false;
                    rare_a = !self_a;
                    rare_b = CJ == 8 && !self_b;
                } else {
                    in_a = L.d2a < lo && !self_a, in_b = L.d2b < lo && !self_b;
                    rare_a = !in_a && !(L.d2a > hi_t) && !self_a;
                    rare_b = !in_b && !(L.d2b > hi_t) && !self_b;
                }
                if (LJ) {
                    rare_a = rare_a || (in_a && L.d2a < close2);
                    rare_b = rare_b || (in_b && L.d2b < close2);
                    in_a = in_a && !(L.d2a < close2);
                    in_b = in_b && !(L.d2b < close2);
                }
                if (rare_a | rare_b) {
                    double* side = &s_side[i_local][0];
                    const uint64_t jb = uint64_t(S.idx[e]) * CJ;
                    if (rare_a && jb + jq < A.n) {
                        const int rc = rare_slot<K>(A, i, jb + jq, r2, side);
                        cnt += rc > 0, coincident |= rc < 0;
                    }
                    if (rare_b && jb + jq + 4 < A.n) {
                        const int rc = rare_slot<K>(A, i, jb + jq + 4, r2, side);
                        cnt += rc > 0, coincident |= rc < 0;
                    }
                }
                cnt += uint32_t(in_a) + uint32_t(in_b);
                if (K == SFCNL_KERNEL_DENSITY) {
                    // cubic spline W(q)/sigma = 2 max(1-q,0)^3 - 8 max(1/2-q,0)^3
                    // (= 1 + 6q^2(q-1) for q <= 1/2, 2(1-q)^3 for 1/2 < q <= 1)
                    const f2 q = f2mul(f2p(sqrt_ftz(L.d2a), sqrt_ftz(L.d2b)), invh2);
                    float q0, q1;
                    f2u(q, q0, q1);
                    const f2 t = f2p(fmaxf(1.f - q0, 0.f), fmaxf(1.f - q1, 0.f));
                    const f2 u = f2p(fmaxf(0.5f - q0, 0.f), fmaxf(0.5f - q1, 0.f));
                    const f2 t3 = f2mul(f2mul(t, t), t), u3 = f2mul(f2mul(u, u), u);
                    const f2 wv = f2fma(f2p(-8.f, -8.f), u3, f2mul(f2p(2.f, 2.f), t3));
                    acc0 = f2fma(f2p(in_a ? L.pma : 0.f, in_b ? L.pmb : 0.f), wv, acc0);
                } else if (LJ) {
                    const f2 inv2 = f2p(in_a ? rcp_ftz(L.d2a) : 0.f, in_b ? rcp_ftz(L.d2b) : 0.f);
                    const f2 s2 = f2mul(f2p(sig2, sig2), inv2);
                    const f2 s6 = f2mul(f2mul(s2, s2), s2);
                    const f2 coef = f2mul(f2mul(f2mul(f2p(eps24, eps24), inv2), s6),
                                          f2fma(f2p(2.f, 2.f), s6, f2p(-1.f, -1.f)));
                    f2 ee = f2mul(f2mul(f2p(eps4, eps4), s6), f2sub(s6, f2p(1.f, 1.f)));
                    f2 cf = coef;
                    if (K == SFCNL_KERNEL_LJ_COULOMB) {
                        const uint64_t jb = uint64_t(S.idx[e]) * CJ;
                        const float qi = float(A.ck * A.q[i]);
                        const float qa = in_a ? qi * float(A.q[jb + jq]) : 0.f;
                        const float qb = (CJ == 8 && in_b) ? qi * float(A.q[jb + jq + 4]) : 0.f;
                        float ra, rb;
                        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(L.d2a));
                        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(L.d2b));
                        const f2 qr = f2mul(f2p(qa, qb), f2p(ra, rb));
                        ee = f2add(ee, qr);
                        cf = f2fma(qr, inv2, cf);
                    }
                    acc0 = f2fma(cf, L.dx, acc0);
                    acc1 = f2fma(cf, L.dy, acc1);
                    acc2 = f2fma(cf, L.dz, acc2);
                    acc3 = f2add(acc3, ee);
                }
            };
            const int self_lo = int(p0) - (CJ - 1);  // j-clusters overlapping [p0, p0 + 64)
            for (uint32_t g = 0; g < n; g += 32) {
                const bool have = g + lane < n;
                const bool mb = have && ((S.msk[g + lane] >> warp) & 1u);
                const int jf = have ? int(S.idx[g + lane]) * CJ - self_lo : -1;
                const unsigned selfm = __ballot_sync(0xffffffffu, jf >= 0 && jf < kSC + CJ - 1);
                unsigned mine = __ballot_sync(0xffffffffu, mb);
                if (unsafe) {
                    while (mine) {
                        const uint32_t e = g + __ffs(mine) - 1;
                        mine &= mine - 1;
                        compute(e, load(e), BoolC<true>(), BoolC<true>());
                    }
                    continue;
                }
                unsigned ms = mine & selfm;
                mine &= ~selfm;
                while (mine) {
                    const uint32_t e1 = g + __ffs(mine) - 1;
                    mine &= mine - 1;
                    if (!LJ && mine) {  // two entries in flight (register budget allows it for density)
                        const uint32_t e2 = g + __ffs(mine) - 1;
                        mine &= mine - 1;
                        const Ld L1 = load(e1), L2 = load(e2);
                        compute(e1, L1, BoolC<false>(), BoolC<false>());
                        compute(e2, L2, BoolC<false>(), BoolC<false>());
                    } else {
                        compute(e1, load(e1), BoolC<false>(), BoolC<false>());
                    }
                }
                while (ms) {
                    const uint32_t e = g + __ffs(ms) - 1;
                    ms &= ms - 1;
                    compute(e, load(e), BoolC<true>(), BoolC<false>());
                }
            }
        }
        const bool last = M.last;
        const uint64_t sc = M.sc;
        if (last) {
            __syncwarp();  // this warp's s_side rows complete
            if (coincident) raise_error(A.err, sc, SFCNL_INPUT_ERROR, kMsgCoincident, 0);
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
            if (active && jq == 0 && !bad) {
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
        }
        nbar_arrive(3 + buf, kWsThreads);  // EMPTY[buf]
        buf ^= 1;
        if (last && sc + gridDim.x >= A.num_sc) break;
    }
}

template <int K, int CJ>
size_t ws_smem() {
    return 2 * sizeof(WsStage<K>);
}
