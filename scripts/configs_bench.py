# Per-stage times of one device-resident step for the BASELINE configs C2, C3, C4 (one B200).
import sys, json
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
cfgs = {
    "C2 uniform 2^26": ("uniform", 1 << 26, dict(density=float(1 << 26), target_neighbors=200.0), 1.0, 0.5 * (1.0 / (1 << 26)) ** (1 / 3)),
    "C3 evrard 2^24": ("evrard", 1 << 24, dict(target_neighbors=200.0), 1.0, 0.5 * (1.0 / (1 << 24)) ** (1 / 3)),
    "C4 LJ fluid 4M skin": ("uniform", 4_000_000, dict(density=100.0, target_neighbors=150.0), 1.100642, 0.2),
}
for name, (gen, n, kw, scale, sigma) in cfgs.items():
    ctx = S.Context(0)
    ps, box = (S.make_uniform(S.UniformSpec(n=n, seed=42, **kw)) if gen == "uniform"
               else S.make_evrard(S.EvrardSpec(n=n, seed=42, **kw)))
    bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, scale)
    pipe = S.Pipeline(ctx, ps, box, bp, [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)], S.PassConfig(1.0, S.MIXED))
    pipe.upload()
    for _ in range(2):
        pipe.run()
    ctx.synchronize()
    ctx.set_timing(True)
    ctx.sort(pipe.bits); ctx.apply_order(); ctx.octree(pipe.bucket); nsc, nb = ctx.build_store(bp)
    st = {k: round(v, 2) for k, v in ctx.stage_times().items() if k != "pass"}
    for k in pipe.kernels:
        ctx.reduce(k, pipe.cfg, n, download=False)
        st["pass_" + k.names[0]] = round(ctx.stage_times()["pass"], 2)
    ctx.set_timing(False)
    tot = sum(st.values())
    print(json.dumps({"config": name, "n": n, "total_ms": round(tot, 2), "ns_per_particle": round(tot * 1e6 / n, 3),
                      "bytes_per_particle": round((nb + 12 * nsc) / n, 4), "stages_ms": st}), flush=True)
    del pipe, ctx
