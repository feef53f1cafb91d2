"""Benchmark: neighbor-list build + neighborhood pass (BASELINE.json metric).

One step = the reference's build-and-query sequence on one batch of particles
(bench.cpp:147-186, with every stage timed, including the sort/permute/octree
that run_bench leaves out): sort_by_sfc -> apply_sfc_order -> build_octree ->
build_neighbor_store -> reduce(SPH density) -> reduce(Lennard-Jones).

Workload (BASELINE.json configs[1], "C2"): 2^26 uniform random particles per GPU in
a periodic unit cube, h for ~200 neighbours, ClusterParams(8,8,32), gather,
compressed; LJ sigma = 0.5 * N^-1/3 (bench.cpp:73-74); mixed-precision pass
(exact pair set, values within 1e-5). Inputs (2.7 GB) exceed L2 (126 MB).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--n N]

Multi-GPU (torchrun, N > 1): SFC key-range domain decomposition
(paper_2602_19873_b200/distributed.py). The global set is N x 2^26
uniform particles in the periodic unit cube (h for 200 neighbours at the global
density); every rank starts from its own 2^26 (spatially random) particles, and one
step = exact distributed split + particle all-to-all + global octree + node-geometry
all-reduce + halo exchange + range build + density + LJ on the rank's super-clusters
(weak scaling; NCCL over NVLink). The step time is the max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ns/particle for list build + neighborhood pass (SPH density + LJ)"
UNIT = "ns/particle"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--particles", "--n", dest="n", type=int, default=1 << 26)  # per GPU
    p.add_argument("--target", type=float, default=200.0)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--cpu-sample", type=int, default=1 << 20)  # cpu_baseline leg of the b200 arm
    p.add_argument("--ref-n", type=int, default=0)  # --impl reference: particles (0 = the full workload)
    p.add_argument("--no-f64", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 or os.environ.get("SFCNL_BENCH_FORCE_DIST"):
        import torch
        import torch.distributed as dist
        backend = os.environ.get("SFCNL_BENCH_BACKEND", "nccl")  # gloo: several ranks on one GPU (testing)
        if backend != "nccl":
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return ws, rank, local


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def composite_roofline(stage, n, pk, ms):
    """sum over stages of the time the stage's binding resource needs for
    its algorithmic work, over the measured step. Streaming stages are bound by HBM
    (compulsory bytes per particle); the build and the passes by the FP32 lanes
    (148 SMs x 128 lanes x 1.965 GHz = 37.2 T lane-ops/s; algorithmic lane-ops per
    particle from the reference's measured work counters: build 464 pair tests x 9,
    density 644 slots x 18 + 200 hits x 12, LJ 644 slots x 12 (hi+lo d2) + 200 hits x 16)."""
    bw = pk["hbm_gbs"] * 1e9
    lane_ops = 148 * 128 * 1.965e9
    hbm_bytes = {"keygen": 36, "sort": 24 * ((3 * 21 + 7) // 8), "permute": 84, "octree": 11,
                 "node_geometry": 14, "cluster_geometry": 46, "encode": 3.77}
    alu_ops = {"build": 464 * 9, "pass_rho": 644 * 18 + 200 * 12, "pass_fx": 644 * 12 + 200 * 16}
    floor = {k: v * n / bw * 1e3 for k, v in hbm_bytes.items() if k in stage}
    floor.update({k: v * n / lane_ops * 1e3 for k, v in alu_ops.items() if k in stage})
    tot = sum(floor.values())
    return {"frac": round(tot / ms, 4), "floor_ms": round(tot, 2),
            "stage_frac": {k: round(floor[k] / stage[k], 3) for k in floor if stage.get(k, 0) > 0},
            "model": "HBM bytes for streaming stages, FP32 lane-ops for build/passes (bench.py composite_roofline)"}


# FP32 lane-ops per unit of work (SURVEY §8(d) cost model): per pair slot the
# d2 (and for LJ the hi+lo correction) + masks, per in-range pair the kernel value
LANE_OP_MODEL = {
    "pass_fx": "12 per pair slot (hi+lo d2: 9, mask 3) + 16 per in-range pair (rcp, s6, coef, energy, 4 sums)",
    "pass_rho": "18 per pair slot (d2 6, sqrt, spline 10, mask) + 12 per in-range pair",
    "build": "9 per exact pair test (464 per particle, neighbor_build.cpp:128-161)",
}


def lane_ops(kernel, slots, hits, n):
    if kernel == "pass_fx":
        return 12 * slots + 16 * hits
    if kernel == "pass_rho":
        return 18 * slots + 12 * hits
    if kernel == "build":
        return 9 * 464 * n
    return None


# ---------------------------------------------------------------- CPU reference
def cpu_reference(n, target, steps=1):
    """The unmodified reference (oracle/_ref) on all host threads; every stage timed."""
    from oracle.oracle import Oracle
    import ctypes as C
    R = Oracle("reference")
    ps = R.make_uniform(n, float(n), target, (1, 1, 1), 0.0, 42)
    threads = os.cpu_count() or 1
    sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
    times = []
    per = (C.c_int * 3)(1, 1, 1)
    D = C.c_double
    stages = None
    for _ in range(steps):
        t = (C.c_double * 7)()
        st = (C.c_double * 4)()
        rc = R.lib.ref_pipeline(C.c_uint64(n), *(a.ctypes.data_as(C.POINTER(D)) for a in (ps.x, ps.y, ps.z, ps.h, ps.m)),
                                ps.box6.ctypes.data_as(C.POINTER(D)), per, C.c_uint32(8), C.c_uint32(8), C.c_int(32),
                                D(1.0), C.c_int(threads), D(1.0), D(sigma), C.c_int(1), t, st, None)
        R._check(rc)
        times.append(t[6])
        stages = {k: t[i] for i, k in enumerate(["sort_by_sfc", "apply_sfc_order", "build_octree",
                                                 "build_neighbor_store", "reduce_density", "reduce_lj", "total"])}
    ms = float(np.median(times))
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), model)
    except OSError:
        pass
    return {"value": ms * 1e6 / n, "unit": UNIT, "cores": threads, "kind": "reference", "cpu_model": model,
            "sample": f"uniform {n} particles (same density/h for {target:.0f} nbrs), full build + density + LJ, "
                      f"median of {steps}", "stages_ms": stages, "bytes_per_particle": st[0]}


def run_reference(args, ws, rank):
    """The unmodified reference on the host cores, on the SAME workload as the b200 arm
    (C2: 2^26 particles per GPU, build + density + LJ). One full-size step takes about two
    minutes on 16 threads, so the arm times ONE step after a small warm-up sample (page-in
    of the library and the thread pool); --ref-n overrides the size."""
    if rank != 0:
        return
    n = args.ref_n or args.n
    t0 = time.time()
    if args.warmup:
        cpu_reference(min(n, 1 << 18), args.target, 1)
    res = cpu_reference(n, args.target, 1)
    out = {"metric": METRIC, "value": res["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": 1, "warmup": args.warmup, "ms_per_step": res["value"] * n / 1e6,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference make_uniform, seed 42)",
           "config": {"workload": "C2 uniform periodic, 200 nbrs, 8x8 gather compressed, build+density+LJ",
                      "n_per_gpu": args.n, "sample_n": n, "same_config": n == args.n},
           "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")},
           "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "stages_ms": res["stages_ms"], "wall_s": round(time.time() - t0, 1)}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- B200 arm
_TORCH_DT = {}


def run_b200(args, ws, rank, local):
    import torch
    _TORCH_DT.update({np.dtype(np.uint32): torch.int32, np.dtype(np.uint64): torch.int64,
                      np.dtype(np.uint8): torch.uint8, np.dtype(np.float64): torch.float64})
    import paper_2602_19873_b200 as S

    n = args.n
    ctx = S.Context(local)
    spec = S.UniformSpec(n=n, density=float(n), target_neighbors=args.target, seed=42 + rank)
    ps, box = S.make_uniform(spec)
    # pinned host buffers for the end-to-end leg
    pinned = {}
    for name in ("x", "y", "z", "h"):
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = getattr(ps, name)
        pinned[name] = t
    t = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = ps.fields["m"]
    pinned["m"] = t
    pps = S.ParticleSet(pinned["x"].numpy(), pinned["y"].numpy(), pinned["z"].numpy(), pinned["h"].numpy(),
                        {"m": pinned["m"].numpy()})
    sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
    kernels = [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)]
    bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0)
    pipe = S.StreamedPipeline(ctx, pps, box, bp, kernels, S.PassConfig(1.0, S.MIXED))
    pipe.upload()
    # pinned host result buffers for the end-to-end leg (a serving loop reuses them)
    pipe.host_buffers(lambda cnt, dt: torch.empty(int(cnt), dtype=_TORCH_DT[np.dtype(dt)], pin_memory=True).numpy().view(dt))
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    for _ in range(args.warmup):
        pipe.run()
    ctx.synchronize()
    # per-stage breakdown from one instrumented step (not part of the timed steps)
    ctx.set_timing(True)
    stage = {}
    ctx.sort(pipe.bits)
    ctx.apply_order()
    ctx.octree(pipe.bucket)
    ctx.build_store(bp)
    st = ctx.stage_times()
    stage.update({k: v for k, v in st.items() if k != "pass"})
    for k in kernels:
        ctx.reduce(k, pipe.cfg, n, download=False)
        stage["pass_" + k.names[0]] = ctx.stage_times()["pass"]
    # fp64 (bit-exact, = reduce<double>) passes over the same store, for the secondary line
    if not args.no_f64:
        for k in kernels:
            ctx.reduce(k, S.PassConfig(1.0, S.F64), n, download=False)
            stage["f64_" + k.names[0]] = ctx.stage_times()["pass"]
    ctx.set_timing(False)
    # work counters of this store for the FP32 lane-op roofline: pair slots (cluster_overhead
    # numerator, bench.cpp:93-122) and in-range pairs (sum of LJ neighbour counts)
    slots = ctx.cluster_slots()
    ctx.reduce(kernels[1], pipe.cfg, n, download=False)
    hits = int(ctx.device_array("count", torch.int32, n).to(torch.int64).sum().item())

    barrier(ws)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            pipe.run()
        ev1.record(stream)
        ev1.synchronize()
    ctx.synchronize()
    barrier(ws)
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launch_count() - launches0) // args.steps
    ms_max = allreduce_max(ms, ws)
    value_job = ms_max * 1e6 / (n * ws)  # whole job: ws*n particles processed in ms_max

    # end-to-end through the C-ABI with host (pinned) buffers
    e2e_ms = []
    for _ in range(args.e2e_steps):  # one step at a time, transfers serialised with the step
        ctx.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        pipe.run_e2e()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_sync = allreduce_max(float(np.median(e2e_ms)) if e2e_ms else float("nan"), ws)
    # streamed: K consecutive steps, each uploading its inputs and downloading its
    # results, with the transfers overlapped with the neighbouring steps' device work
    e2e = float("nan")
    k_stream = max(16, 8 * args.e2e_steps) if args.e2e_steps > 0 else 0
    if k_stream:
        pipe.run_stream(2)  # warm-up: side buffers allocated once
        ctx.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        pipe.run_stream(k_stream)
        e2e = allreduce_max((time.perf_counter() - t0) * 1e3 / k_stream, ws)

    bpp = (pipe.blob_bytes + 4 * pipe.num_sc + 8 * (pipe.num_sc + 1)) / n
    pk, pk_kind = peaks()
    stage_mixed = {k: v for k, v in stage.items() if not k.startswith("f64_")}
    # dominant kernel + its algorithmic bytes
    algo_bytes = {
        "build": 32 + 8 + 3.77,            # sorted x,y,z,h read + node/cluster geo (amortised) + store write
        "pass_rho": 32 + 8 + 3.77 + 12,    # i x,y,z,h + j m + list + rho/count written
        "pass_fx": 32 + 3.77 + 36,         # i x,y,z,h + list + 4 outputs + count written
        "sort": 24 * ((3 * 21 + 7) // 8),
    }
    dom = max(stage_mixed, key=lambda k: stage_mixed[k])
    dom_ms = stage_mixed[dom]
    ab = algo_bytes.get(dom, 48.0) * n
    achieved = ab / (dom_ms * 1e-3) / 1e9
    # FP32 lane-op roofline of the dominant kernel: algorithmic lane-ops per
    # launch from this store's own work counters, over the measured launch time; peak = every
    # FP32 lane of the part busy every cycle (148 SMs x 128 lanes x max SM clock)
    ops = lane_ops(dom, slots, hits, n)
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    peak_t = 148 * 128 * sm_mhz * 1e6 / 1e12
    achieved_t = ops / (dom_ms * 1e-3) / 1e12 if ops else None
    traffic, pipe_util, cap = None, None, None
    try:  # DRAM bytes and pipe utilisation of the same kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as f:
            tj = json.load(f)
        if int(tj["n"]) == n:
            traffic = tj["dram_bytes_per_launch"].get(dom)
            pipe_util = tj["pipe_util_pct"].get(dom)
            cap = tj.get("capture")
    except (OSError, KeyError, ValueError):
        pass
    out = {
        "metric": METRIC, "value": round(value_job, 4), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "mixed f32/f64 (exact f64 cutoff decisions)",
        "data": "synthetic (make_uniform, seed 42+rank)",
        "config": {"workload": ("C2: 2^26" if n == 1 << 26 else f"C2-shaped: {n}") +
                               " uniform periodic unit cube per GPU, 200 nbrs, ClusterParams(8,8,32) "
                               "gather compressed, build + SPH density + LJ (mixed)",
                   "n_per_gpu": n, "global_particles": n * ws,
                   "l2": f"inputs {n * 40 / 1e9:.2f} GB " + ("> L2, no flush" if n * 40 > 126e6 else "(fits L2)"),
                   "bytes_per_particle": round(bpp, 4), "parallelism": f"domain-replica x{ws}"},
        "e2e": {"value": round(e2e * 1e6 / n, 4), "unit": UNIT, "ms_per_step": round(e2e, 2),
                "h2d_bytes_per_step": pipe.h2d_bytes(), "d2h_bytes_per_step": pipe.d2h_bytes(),
                "mode": f"streamed over {k_stream} steps: every step's pinned-host H2D of its inputs and D2H of its "
                        "store + pass outputs, overlapped with the neighbouring steps' device work",
                "serialised_ms_per_step": round(e2e_sync, 2)},
        "gpu_launches": int(launches),
        "stages_ms": {k: round(v, 3) for k, v in stage_mixed.items()},
        "f64": ({"ms_per_step": round(ms_max - stage["pass_rho"] - stage["pass_fx"] + stage["f64_rho"] + stage["f64_fx"], 3),
                 "pass_rho_ms": round(stage["f64_rho"], 3), "pass_fx_ms": round(stage["f64_fx"], 3),
                 "note": "same step with the bit-exact fp64 passes (= reduce<double>) instead of the mixed ones"}
                if "f64_rho" in stage else None),
        "roofline": {"bound": "fp32", "kernel": dom,
                     "achieved": round(achieved_t, 3) if achieved_t else None, "peak": round(peak_t, 2),
                     "unit": "TFLOP/s", "frac": round(achieved_t / peak_t, 4) if achieved_t else None,
                     "traffic": traffic, "traffic_capture": cap, "pipe_util_pct": pipe_util,
                     "work": {"pair_slots": int(slots), "in_range_pairs": hits, "lane_ops": ops,
                              "model": LANE_OP_MODEL.get(dom)},
                     "note": "FP32 lane-ops (one per FADD/FMUL/FFMA lane), peak = 148 SMs x 128 FP32 lanes x max SM "
                             "clock; the build and passes are FP32-issue bound (SURVEY §8(d))",
                     "hbm": {"achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                             "frac": round(achieved / pk["hbm_gbs"], 4), "peak_kind": pk_kind,
                             "algorithmic_bytes_per_particle": algo_bytes.get(dom)}},
        "roofline_composite": composite_roofline(stage_mixed, n, pk, ms_max),
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference(args.cpu_sample, args.target, 1)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
            out["cpu_baseline"]["stages_ms"] = cb["stages_ms"]
        except Exception as e:  # the checker library is absent
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_b200_distributed(args, ws, rank, local):
    import torch
    import paper_2602_19873_b200 as S
    from paper_2602_19873_b200.distributed import Comm, CudaEngine, DomainDecomposition

    n = args.n
    ctx = S.Context(local)
    # rank's share of a global uniform set of ws*n particles in the unit cube
    ps, _ = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=args.target, seed=42 + rank))
    ps.h[:] = S.uniform_h_for_target(args.target, float(n * ws))
    box = S.SimulationBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (True, True, True))
    pinned = {}
    for name, v in (("x", ps.x), ("y", ps.y), ("z", ps.z), ("h", ps.h), ("m", ps.fields["m"])):
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = v
        pinned[name] = t
    pps = S.ParticleSet(pinned["x"].numpy(), pinned["y"].numpy(), pinned["z"].numpy(), pinned["h"].numpy(),
                        {"m": pinned["m"].numpy()})
    sigma = 0.5 * (1.0 / (n * ws)) ** (1.0 / 3.0)
    kernels = [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)]
    bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0)
    E = CudaEngine(ctx, box, ["m"])
    E.upload(pps)
    dd = DomainDecomposition(E, Comm(), bp, kernels, S.PassConfig(1.0, S.MIXED))
    for _ in range(args.warmup):
        res = dd.run(download=False)
    ctx.synchronize()
    barrier(ws)
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(E.stream)
        for _ in range(args.steps):
            res = dd.run(download=False)
        ev1.record(E.stream)
        ev1.synchronize()
    ctx.synchronize()
    barrier(ws)
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launch_count() - launches0) // args.steps
    ms_max = allreduce_max(ms, ws)
    value_job = ms_max * 1e6 / (n * ws)
    # end to end: pinned host inputs -> step -> store + outputs back to the host
    e2e_ms, rr = [], None
    for _ in range(args.e2e_steps):
        ctx.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        E.upload(pps)
        rr = dd.run(download=True)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e = allreduce_max(float(np.median(e2e_ms)) if e2e_ms else float("nan"), ws)
    nloc = res.p_end - res.p_begin
    d2h = 0
    if rr is not None:
        d2h = rr.store.total_bytes() + sum(12 * nloc if len(k.names) == 1 else 36 * nloc for k in kernels)
    halo = allreduce_max(float(res.halo_particles), ws)
    # stage times of one instrumented step (build = dominant kernel), for the roofline
    ctx.set_timing(True)
    dd.run(download=False)
    st = ctx.stage_times()
    ctx.set_timing(False)
    pk, pk_kind = peaks()
    b_ms = st.get("build", float("nan"))
    achieved = (32 + 8 + 3.77) * nloc / (b_ms * 1e-3) / 1e9 if b_ms > 0 else None
    out = {
        "metric": METRIC, "value": round(value_job, 4), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "mixed f32/f64 (exact f64 cutoff decisions)",
        "data": "synthetic (make_uniform per rank, seed 42+rank, global density)",
        "config": {"workload": f"C2 weak-scaled: {ws} x " + ("2^26" if n == 1 << 26 else str(n)) + " uniform periodic unit cube, 200 nbrs, "
                               "ClusterParams(8,8,32) gather compressed, build + SPH density + LJ (mixed)",
                   "n_per_gpu": n, "global_particles": n * ws, "l2": "inputs 2.7 GB/GPU > L2, no flush",
                   "parallelism": f"sfc-domain x{ws} (NCCL all-to-all + halo)",
                   "max_halo_particles_per_rank": int(halo)},
        "e2e": {"value": round(e2e * 1e6 / (n * ws), 4) if e2e == e2e else None, "unit": UNIT,
                "ms_per_step": round(e2e, 2), "h2d_bytes_per_step": 40 * n, "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "stages_ms_last_call": {k: round(v, 3) for k, v in st.items()},
        "roofline": {"bound": "hbm", "kernel": "build", "achieved": round(achieved, 1) if achieved else None,
                     "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None, "traffic": None,
                     "peak_kind": pk_kind},
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif ws > 1 or os.environ.get("SFCNL_BENCH_FORCE_DIST"):
        run_b200_distributed(args, ws, rank, local)
    else:
        run_b200(args, ws, rank, local)
    if ws > 1 or os.environ.get("SFCNL_BENCH_FORCE_DIST"):
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
