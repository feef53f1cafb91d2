"""SFC domain decomposition: P ranks, each building and querying only its
own super-clusters, must reproduce the single-domain store byte for byte and the
single-domain pass outputs exactly (fp64 gather mode).

CPU: world_size 2 and 3 over gloo with the oracle engine (tests/dist_engines.py).
GPU: world_size 2 over gloo with two ranks sharing cuda:0 through the C-ABI engine.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402

from paper_2602_19873_b200.distributed import sc_partition  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(world, cfg, tmp_path, timeout=600):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", LOCAL_WORLD_SIZE=str(world),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), str(tmp_path),
                                       json.dumps(cfg)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=timeout)
            outs.append(out.decode(errors="replace"))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


def single_domain(cfg):
    o = Oracle("port")
    if cfg.get("dist", "uniform") == "uniform":
        gp = o.make_uniform(cfg["n"], float(cfg["n"]), cfg["target"], tuple(cfg["periodic"]),
                            cfg.get("h_jitter", 0.0), cfg["seed"])
    else:
        gp = o.make_evrard(cfg["n"], cfg["target"], False, tuple(cfg["periodic"]), cfg["seed"])
    keys, perm, sp, tree, store = o.pipeline(gp, ci=cfg["ci"], cj=cfg["cj"], w=cfg["w"], mode=cfg.get("mode", 0),
                                             scale=cfg.get("scale", 1.0))
    single_domain.tree = tree
    eps_sig = {"lj": (1.0, 0.05, 0.0), "lj_coulomb": (1.0, 0.05, 0.3)}
    outs = []
    for k in cfg["kernels"]:
        e, s, ck = eps_sig.get(k, (1.0, 1.0, 0.0))
        outs.append(o.reduce(k, sp, store, cfg.get("query_scale", 1.0), e, s, ck))
    return store, outs


def check(parts, cfg, exact=True):
    store, outs = single_domain(cfg)
    n = cfg["n"]
    scb, pb = sc_partition(n, len(parts))
    for r, p in enumerate(parts):
        assert (int(p["p0"]), int(p["p1"]), int(p["sc0"]), int(p["sc1"])) == (pb[r], pb[r + 1], scb[r], scb[r + 1])
    counts = np.concatenate([p["counts"] for p in parts])
    assert np.array_equal(counts, store.counts)
    blob = np.concatenate([p["blob"] for p in parts])
    assert np.array_equal(blob, store.blob)
    base, offs = 0, []
    for p in parts:
        offs.append(p["offsets"][:-1].astype(np.uint64) + np.uint64(base))
        base += len(p["blob"])
    assert np.array_equal(np.concatenate(offs + [np.array([base], np.uint64)]), store.offsets)
    for k, (ref_outs, ref_cnt) in enumerate(outs):
        cnt = np.concatenate([p[f"k{k}_cnt"] for p in parts])
        assert np.array_equal(cnt, ref_cnt)
        for j, ref in enumerate(ref_outs):
            got = np.concatenate([p[f"k{k}_o{j}"] for p in parts])
            if exact:
                assert np.array_equal(got, ref), (k, j)
            else:
                assert np.allclose(got, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max()), (k, j)
    assert len(parts) == 1 or all(int(p["halo"]) > 0 for p in parts)  # one rank: no halo
    t = single_domain.tree
    for p in parts:  # every rank holds the single-domain octree (distributed build)
        if "t_kf" in p:
            for a, b in (("t_kf", t.key_first), ("t_kl", t.key_last), ("t_pb", t.pbegin), ("t_pe", t.pend),
                         ("t_fc", t.first_child), ("t_d", t.depth)):
                assert np.array_equal(p[a], b), a


CPU_CASES = [
    dict(n=6000, target=40, periodic=[1, 1, 1], seed=5, ci=8, cj=8, w=32, kernels=["density", "count"]),
    dict(n=5000, target=30, periodic=[1, 0, 1], seed=9, ci=8, cj=4, w=64, h_jitter=0.3, kernels=["lj"]),
    dict(n=4000, target=40, periodic=[0, 0, 0], seed=2, ci=8, cj=8, w=32, dist="evrard", kernels=["density"]),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", range(len(CPU_CASES)))
def test_domain_decomposition_oracle_engine(tmp_path, world, case):
    cfg = dict(CPU_CASES[case], engine="oracle")
    check(launch(world, cfg, tmp_path), cfg)


def test_domain_decomposition_one_rank_collectives_issued(tmp_path, monkeypatch):
    """World size 1 with every collective issued (SFCNL_COMM_ALWAYS=1; the GPU twin of
    this test runs it over NCCL) equals the single-domain run."""
    monkeypatch.setenv("SFCNL_COMM_ALWAYS", "1")
    cfg = dict(CPU_CASES[0], engine="oracle")
    check(launch(1, cfg, tmp_path), cfg)


def test_domain_decomposition_legacy_orchestration(tmp_path, monkeypatch):
    """The global-index orchestration (symmetric stores use it) on the oracle engine."""
    monkeypatch.setenv("SFCNL_DD_LEGACY", "1")
    cfg = dict(CPU_CASES[0], engine="oracle")
    check(launch(2, cfg, tmp_path), cfg)


GPU_CASES = [
    dict(n=40000, target=60, periodic=[1, 1, 1], seed=11, ci=8, cj=8, w=32, kernels=["density", "lj"]),
    dict(n=12000, target=40, periodic=[1, 1, 0], seed=8, ci=1, cj=1, w=32, h_jitter=0.2, kernels=["density", "lj_coulomb"]),
    dict(n=30000, target=50, periodic=[0, 0, 0], seed=4, ci=8, cj=4, w=64, dist="evrard", kernels=["density"]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GPU_CASES)))
def test_domain_decomposition_cuda_engine_fp64(tmp_path, case):
    cfg = dict(GPU_CASES[case], engine="cuda", precision=0)
    check(launch(2, cfg, tmp_path), cfg)


SYM_CASES = [
    dict(n=30000, target=50, periodic=[1, 1, 1], seed=7, ci=8, cj=8, w=32, mode=1, h_jitter=0.3,
         kernels=["density", "lj", "count", "lj_coulomb"]),
    dict(n=20000, target=40, periodic=[0, 0, 0], seed=3, ci=8, cj=4, w=64, mode=1, dist="evrard", kernels=["density"]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", range(len(SYM_CASES)))
def test_domain_decomposition_symmetric_fp64(tmp_path, world, case):
    """Symmetric stores: the reverse halo reduction keeps the reference's global entry
    order, so the distributed outputs are bit-equal to the single-domain reduce<double>."""
    cfg = dict(SYM_CASES[case], engine="cuda", precision=0)
    check(launch(world, cfg, tmp_path), cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [0, 2])
def test_domain_decomposition_nccl_one_rank(tmp_path, monkeypatch, case):
    """The NCCL branch of Comm (device tensors: all_reduce SUM/MIN/MAX,
    all_gather_into_tensor, all_to_all_single with split sizes) on the one GPU this
    harness has: a world-1 NCCL group with the collectives issued instead of
    short-circuited (SFCNL_COMM_ALWAYS=1) reproduces the single-domain run."""
    monkeypatch.setenv("SFCNL_COMM_ALWAYS", "1")
    cfg = dict(GPU_CASES[case], engine="cuda", precision=0, backend="nccl")
    check(launch(1, cfg, tmp_path), cfg)


@pytest.mark.gpu
def test_domain_decomposition_cuda_engine_mixed(tmp_path):
    cfg = dict(GPU_CASES[0], engine="cuda", precision=1, kernels=["density", "count"])
    check(launch(2, cfg, tmp_path), cfg, exact=False)


@pytest.mark.gpu
def test_range_build_and_pass_slices_single_gpu():
    """build_store_range / reduce over super-cluster ranges of a complete particle set
    equal the corresponding slices of the whole-set store and outputs."""
    import paper_2602_19873_b200 as sfcnl
    ps, box = sfcnl.make_uniform(sfcnl.UniformSpec(n=50000, density=50000.0, target_neighbors=80, seed=3))
    ctx = sfcnl.Context(0)
    order = sfcnl.sort_by_sfc(ps, box, ctx=ctx)
    tree = sfcnl.build_octree(order, ctx=ctx)
    sps = sfcnl.apply_sfc_order(ps, order, ctx=ctx)
    bp = sfcnl.BuildParams()
    full = sfcnl.build_neighbor_store(sps, box, tree, bp, ctx=ctx)
    cfgs = [sfcnl.PassConfig(1.0, sfcnl.F64), sfcnl.PassConfig(1.0, sfcnl.MIXED)]
    ref = [sfcnl.reduce(sps, box, full, sfcnl.sph_density_kernel(), c, ctx=ctx) for c in cfgs]
    nsc = full.num_superclusters()
    for sc0, sc1 in [(0, 100), (100, 457), (457, nsc), (3, 4), (nsc, nsc)]:
        ctx.set_particles(sps, box, sorted_slot=True)
        ctx.set_octree(tree)
        ns, nb = ctx.build_store_range(bp, sc0, sc1)
        st = ctx.get_store(bp, sps.size(), ns, nb)
        b0, b1 = int(full.offsets[sc0]), int(full.offsets[sc1])
        assert np.array_equal(st.counts, full.counts[sc0:sc1])
        assert np.array_equal(st.blob, full.blob[b0:b1])
        assert np.array_equal(st.offsets, full.offsets[sc0:sc1 + 1] - full.offsets[sc0])
        p0, p1 = min(64 * sc0, sps.size()), min(64 * sc1, sps.size())
        for c, r in zip(cfgs, ref):
            got = ctx.reduce(sfcnl.sph_density_kernel(), c, p1 - p0)
            assert np.array_equal(got.neighbor_count, r.neighbor_count[p0:p1])
            assert np.array_equal(got.outputs[0], r.outputs[0][p0:p1])


@pytest.mark.gpu
def test_domain_decomposition_memory_per_rank(tmp_path):
    """O(N/P): at a simulated world of 8 (eight ranks sharing cuda:0), every rank's device
    allocation for the build + density + LJ step -- its context's buffers plus the torch
    tensors of the orchestration (owned columns, halo rows, index maps), steady state after
    the step -- stays within 1.3x the single-GPU footprint of the same step on the rank's
    own particles. The legacy orchestration allocated every global-index
    array (48 B x N_total per rank) and the whole node geometry."""
    cfg = dict(n=32 << 20, target=200, periodic=[1, 1, 1], seed=21, ci=8, cj=8, w=32, kernels=["density", "lj"],
               engine="cuda", precision=1, measure_memory=True, even_shares=True)
    parts = launch(8, cfg, tmp_path, timeout=1200)
    ratios = []
    for p in parts:
        dd = int(p["dd_ctx"]) + int(p["dd_torch"])
        ratios.append(dd / int(p["single"]))
        print(f"rank single {int(p['single']) / 2**20:.0f} MiB dd {dd / 2**20:.0f} MiB "
              f"(ctx {int(p['dd_ctx']) / 2**20:.0f} + torch {int(p['dd_torch']) / 2**20:.0f}, peak torch "
              f"{int(p['dd_torch_peak']) / 2**20:.0f}) n_in {int(p['n_in'])} n_local {int(p['n_local'])} "
              f"halo {int(p['halo'])}")
    assert max(ratios) <= 1.3, ratios
