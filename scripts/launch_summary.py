"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of scripts/stage_times.py: per kernel launches, time, share,
DRAM bytes; optionally write the per-launch DRAM bytes per stage that bench.py reports
as roofline.traffic (profiles/<round>/traffic.json).
usage: launch_summary.py LAUNCHES.csv N_PARTICLES [TRAFFIC_JSON CAPTURE_NOTE]"""
import collections
import csv
import json
import re
import sys

path, n = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
h = rows[0]
K, ID, M, V = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launch = collections.defaultdict(dict)
for r in rows[1:]:
    launch[(r[ID], r[K])][r[M]] = float(r[V].replace(",", ""))


def short(name):
    name = name.split("(")[0]
    m = re.search(r"(k_\w+)(<.*>)?$", name)
    if not m:
        return name[-40:]
    base, tpl = m.group(1), m.group(2) or ""
    tpl = re.sub(r"unnamed>::|sfcnl_cu::|\(unsigned int\)|\(int\)|\(bool\)", "", tpl)
    return (base + tpl)[:60]


agg = collections.OrderedDict()
for (lid, name), m in sorted(launch.items(), key=lambda kv: int(kv[0][0])):
    a = agg.setdefault(short(name), [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
unit = 1e-6  # ns -> ms
tot = sum(a[1] for a in agg.values())
print(f"# launch list summary, {len(launch)} launches, total {tot * unit:.2f} ms")
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} n={c:3d} {t * unit:9.3f} ms {t / tot * 100:5.1f}%  dram {b / 1e9:8.3f} GB  "
          f"{b / c / n:7.1f} B/particle/launch")

if len(sys.argv) > 3:
    def per_launch(*pats):
        tot_b, cnt = 0.0, 0
        for k, (c, t, b) in agg.items():
            if any(p in k for p in pats):
                tot_b += b
                cnt = max(cnt, c)
        return int(tot_b / max(cnt, 1))

    steps = max(c for k, (c, t, b) in agg.items() if k.startswith("k_keygen"))
    out = {"n": n, "capture": sys.argv[4],
           "dram_bytes_per_launch": {
               "pass_fx": per_launch("k_pass_warp<2"),
               "build": int(sum(b for k, (c, t, b) in agg.items() if "k_build_warp" in k or "k_halo_warp" in k) / steps),
               "pass_rho": per_launch("k_pass_item<1"),
               "sort": per_launch("k_onesweep"),
               "permute": int(sum(b for k, (c, t, b) in agg.items() if "_records" in k) / steps),
               "keygen": per_launch("k_keygen")},
           "pipe_util_pct": {},
           "note": "per-launch DRAM bytes of each stage's kernels at C2 (build = traversal + mask kernel, "
                   "permute = pack + gather)"}
    json.dump(out, open(sys.argv[3], "w"), indent=1)
