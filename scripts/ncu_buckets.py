"""Group SASS instructions of one kernel by execution count (approximates code regions)."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sections, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]; sections.append(cur)
    elif cur is not None:
        cur.append(line)
sec = next(s for s in sections if kern in s[0])
rows = list(csv.reader(sec[1:])); h = rows[0]
IE, SMP = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
b = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[1:]:
    try:
        ie, s = int(r[IE] or 0), int(r[SMP] or 0)
    except (ValueError, IndexError):
        continue
    b[ie][0] += ie; b[ie][1] += s; b[ie][2] += 1
tot = sum(v[0] for v in b.values()); ts = sum(v[1] for v in b.values())
for k, v in sorted(b.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"count {k:>10}  n_instr {v[2]:4d}  exec {v[0]/tot*100:5.1f}%  samples {v[1]/ts*100:5.1f}%")
