"""Debug: CUDA engine steps of the O(N/P) decomposition against the oracle engine, per
rank (launch with torchrun --nproc-per-node 2 on one GPU, gloo)."""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_19873_b200 as S
from paper_2602_19873_b200.distributed import Comm, CudaEngine, DomainDecomposition, sc_partition
from oracle.oracle import Oracle
from dist_engines import OracleEngine
from dist_worker import shares

def _gt_nodes(gt):
    nodes = np.zeros(len(gt.pend), S.api.NODE_DTYPE)
    nodes["key_first"], nodes["key_last"] = gt.key_first, gt.key_last
    nodes["particle_begin"], nodes["particle_end"] = gt.pbegin, gt.pend
    nodes["first_child"], nodes["depth"] = gt.first_child, gt.depth
    return nodes


dist.init_process_group("gloo")
r, P = dist.get_rank(), dist.get_world_size()
o = Oracle("port")
n = 40000
gp = o.make_uniform(n, float(n), 60, (1, 1, 1), 0.0, 11)
b = shares(n, P)
idx = np.arange(b[r], b[r + 1])
box = S.SimulationBox(tuple(gp.box6[:3]), tuple(gp.box6[3:]), (True, True, True))
comm = Comm()
ctx = S.Context(0)
E = CudaEngine(ctx, box, ["m", "q"])
E.upload(S.ParticleSet(gp.x[idx], gp.y[idx], gp.z[idx], gp.h[idx], {"m": gp.m[idx], "q": gp.q[idx]}))
O = OracleEngine(o, gp.box6, gp.periodic)
O.upload(gp.permuted(idx))
keys, perm = o.sort_by_sfc(gp)
gt = o.tree(keys)
with torch.cuda.stream(E.stream):
    k1 = E.local_sort(); k2 = O.local_sort()
    print(r, "local keys equal", np.array_equal(k1.cpu().numpy(), k2.numpy()), flush=True)
    N = n
    scb, pb = sc_partition(N, P); p0, p1 = pb[r], pb[r + 1]
    dd = DomainDecomposition(E, comm, S.BuildParams(), [], S.PassConfig(1.0, S.F64))
    counts = [int(v) for v in comm.all_gather(torch.tensor([int(k1.numel())], dtype=torch.int64, device="cuda")).view(-1).tolist()]
    cut = dd._split(k1, counts, pb)
    ddo = DomainDecomposition(O, comm, S.BuildParams(), [], S.PassConfig(1.0, S.F64))
    cuto = ddo._split(k2, counts, pb)
    print(r, "cut equal", np.array_equal(cut.cpu().numpy(), cuto.numpy()), flush=True)
    nn = E.octree_dist(64, N, comm)
    nd = ctx.get_octree(nn)
    ok = len(nd) == len(gt.pend) and all(np.array_equal(np.asarray(nd[a]).astype(np.int64), getattr(gt, b_).astype(np.int64))
        for a, b_ in (("key_first", "key_first"), ("particle_begin", "pbegin"), ("particle_end", "pend"), ("first_child", "first_child")))
    print(r, "tree equal", ok, nn, len(gt.pend), flush=True)
    cut_h = cut.cpu().numpy()
    send = np.diff(cut_h[r]).tolist(); recv = [int(cut_h[s, r + 1] - cut_h[s, r]) for s in range(P)]
    moved = [comm.all_to_all_v(col, send, recv) for col in E.payload()]
    E.merge_owned(moved, recv)
    sp = gp.permuted(perm)
    print(r, "owned equal", np.array_equal(E.owned[0].cpu().numpy(), sp.x[p0:p1]), np.array_equal(E.owned[3].cpu().numpy(), sp.h[p0:p1]), flush=True)
    lb = E.leaf_boxes(p0, p1).cpu().numpy()
    O.tree = gt; O.owned = sp.permuted(np.arange(p0, p1)); O.n_owned = p1 - p0
    lbo = O.leaf_boxes(p0, p1).numpy()
    print(r, "leaf boxes equal", np.array_equal(lb, lbo), flush=True)
    db = E.domain_boxes(32).cpu().numpy(); dbo = O.domain_boxes(32).numpy()
    print(r, "domain boxes equal", np.allclose(db, dbo), flush=True)
    boxes = comm.all_gather(torch.from_numpy(db).cuda())
    hmax = float(gp.h.max())
    fl = E.halo_select(p0, p1, 8, torch.from_numpy(lbo).cuda(), boxes, r, hmax).cpu().numpy()
    flo = O.halo_select(p0, p1, 8, torch.from_numpy(lbo), boxes.cpu(), r, hmax).numpy()
    print(r, "halo flags equal", np.array_equal(fl, flo), fl.sum(), flo.sum(), flush=True)
    flags = torch.from_numpy(fl).cuda()
    cj = 8; c0 = p0 // cj
    ids = [torch.nonzero(flags[q]).view(-1) + c0 for q in range(P)]
    nsend = torch.tensor([int(t.numel()) for t in ids], dtype=torch.int64, device="cuda")
    mat = comm.all_gather(nsend).cpu().numpy()
    sendc, recvc = mat[r].tolist(), mat[:, r].tolist()
    allids = torch.cat(ids)
    hids = comm.all_to_all_v(allids, sendc, recvc)
    rows = E.pack_clusters(p0, p1, cj, allids)
    hrows = comm.all_to_all_v(rows, [v * cj for v in sendc], [v * cj for v in recvc])
    o_own = E.place_local(N, p0, p1, cj, hids, hrows)
    lpos, present, lc2g = [t.cpu().numpy() for t in E._maps]
    nl = E.n_local
    lx = ctx.get_sorted("x", nl)
    g_of_l = np.full(nl, -1, np.int64)
    for l in range(nl):
        gc = int(lc2g[l // cj]) if l // cj < len(lc2g) else -1
        if gc >= 0 and gc != 0xffffffff and gc != -1:
            g_of_l[l] = gc * cj + l % cj
    ok = g_of_l >= 0
    ok &= g_of_l < N
    print(r, "o_own", o_own, "n_local", nl, "halo", hids.numel(), "local x equal", np.array_equal(lx[ok], sp.x[g_of_l[ok]]),
          "padding NaN", bool(np.isnan(lx[~ok]).all()), flush=True)
    nd = ctx.get_octree(nn)
    lp = lpos.astype(np.int64)
    def mapg(g):
        c = g // cj
        return np.where(c >= len(present), lp[-1], lp[np.minimum(c, len(present) - 1)] * cj + np.where(present[np.minimum(c, len(present) - 1)] > 0, g % cj, 0))
    exp_b = mapg(gt.pbegin.astype(np.int64)); exp_e = np.maximum(mapg(gt.pend.astype(np.int64)), exp_b)
    print(r, "local tree equal", np.array_equal(np.asarray(nd["particle_begin"]).astype(np.int64), exp_b),
          np.array_equal(np.asarray(nd["particle_end"]).astype(np.int64), exp_e), flush=True)
    bp = S.BuildParams()
    st = E.build_range(bp, o_own // 64, o_own // 64 + (scb[r + 1] - scb[r]), hmax, True)
    ref = o.build_store(sp, gt)
    c_ref = ref.counts[scb[r]:scb[r + 1]]
    bad = np.nonzero(st.counts != c_ref)[0]
    print(r, "store counts equal", len(bad) == 0, "first bad", bad[:5], st.counts[bad[:3]], c_ref[bad[:3]], flush=True)
    if len(bad):
        sci = int(bad[0])
        def entries(store, s_):
            c = int(store.counts[s_]); b0, e0 = int(store.offsets[s_]), int(store.offsets[s_ + 1])
            idx_, _ = o.decode(store.blob[b0 + c:e0], c, 32)
            return dict(zip(idx_.tolist(), store.blob[b0:b0 + c].tolist()))
        mine = entries(st, sci); theirs = entries(ref, scb[r] + sci)
        miss = sorted(set(theirs) - set(mine)); extra = sorted(set(mine) - set(theirs))
        diffm = [k for k in set(mine) & set(theirs) if mine[k] != theirs[k]]
        print(r, "SC", sci, "missing", miss[:10], "present?", [int(present[c]) for c in miss[:10]], "extra", extra[:5],
              "mask diffs", diffm[:5], flush=True)
        geo = ctx.node_geometry(nn)
        gq = miss[0] * cj
        # root-to-leaf chain of the global tree containing particle gq
        chain, k = [0], 0
        while gt.first_child[k] >= 0:
            fc = gt.first_child[k]
            k = next(fc + c for c in range(8) if gt.pbegin[fc + c] <= gq < gt.pend[fc + c])
            chain.append(k)
        lsc = o_own // 64 + sci
        igeo = ctx.device_array("cluster_geo.i", torch.float64).view(-1, 8).cpu().numpy()
        scg = igeo[lsc * 8: lsc * 8 + 8]
        sclo, schi, scmh = scg[:, 0:3].min(0), scg[:, 3:6].max(0), scg[:, 6].max()
        L = 1.0
        for k in chain:
            lo, hi = geo[0][k], geo[1][k]
            gap = np.maximum(np.maximum(sclo, lo) - np.minimum(schi, hi), 0)
            gap2 = np.minimum(gap, np.maximum(np.maximum(sclo, lo - L) - np.minimum(schi, hi - L), 0))
            gap2 = np.minimum(gap2, np.maximum(np.maximum(sclo, lo + L) - np.minimum(schi, hi + L), 0))
            print(r, "node", k, "glob", gt.pbegin[k], gt.pend[k], "local", nd[k]["particle_begin"], nd[k]["particle_end"],
                  "box", lo, hi, "d2", float((gap2 ** 2).sum()), "r2", scmh ** 2, flush=True)
        ctx2 = S.Context(0)
        ctx2.set_particles(S.ParticleSet(sp.x, sp.y, sp.z, sp.h, {"m": sp.m}), box, sorted_slot=True)
        ctx2.set_octree(S.Octree(ctx.get_octree(nn) if False else _gt_nodes(gt), 21, N))
        ns2, nb2 = ctx2.build_store_range(bp, scb[r], scb[r + 1], hmax)
        st2 = ctx2.get_store(bp, N, ns2, nb2)
        print(r, "global-array range build equal", np.array_equal(st2.counts, c_ref), flush=True)
    if False:
        geo = ctx.node_geometry(nn)
        # compare local node geometry of leaves fully present with the global
        tg = o.node_geometry(keys, sp)
        lo_g = tg[1]
        leaves = np.nonzero(gt.first_child < 0)[0]
        full = [k for k in leaves if all(present[c] for c in range(gt.pbegin[k] // cj, (gt.pend[k] - 1) // cj + 1)) and gt.pend[k] > gt.pbegin[k]]
        diff = [k for k in full if not np.array_equal(geo[0][k], lo_g[k])]
        print(r, "full leaves", len(full), "geo mismatches", len(diff), diff[:3], flush=True)
        if diff:
            k = diff[0]; print(r, geo[0][k], lo_g[k], nd[k], flush=True)
dist.destroy_process_group()
