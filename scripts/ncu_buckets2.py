"""Sum warp-instructions of one kernel grouped by execution count (loop nests)."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sections, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]; sections.append(cur)
    elif cur is not None:
        cur.append(line)
sec = next(s for s in sections if kern in s[0].replace("(int)", ""))
rows = list(csv.reader(sec[1:])); h = rows[0]
IE, SMP = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
b = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[1:]:
    try:
        c = int(r[IE] or 0); s = int(r[SMP] or 0)
    except ValueError:
        continue
    if c == 0: continue
    k = round(c, -len(str(c)) + 2)
    b[k][0] += c; b[k][1] += 1; b[k][2] += s
tot = sum(v[0] for v in b.values()); ts = sum(v[2] for v in b.values())
for k, v in sorted(b.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"count~{k:>12.3g}  n_instr {v[1]:5d}  warp-instr {v[0]:.3e} ({v[0]/tot*100:5.1f}%)  stall {v[2]/ts*100:5.1f}%")
