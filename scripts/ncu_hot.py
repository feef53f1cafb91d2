"""Summarise an ncu source page (SASS): top instructions by stall samples.
usage: ncu_hot.py REPORT NAME_SUBSTRING [TOP]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sections, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]
        sections.append(cur)
    elif cur is not None:
        cur.append(line)
sec = next(s for s in sections if kern in s[0])
rows = list(csv.reader(sec[1:]))
h = rows[0]
A, S, SMP, IE, AT = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed", "Avg. Threads Executed"))
data = []
for r in rows[1:]:
    try:
        data.append((int(r[IE] or 0), int(r[SMP] or 0), float(r[AT] or 0), r[A][-5:], r[S].strip()))
    except (ValueError, IndexError):
        pass
tot_i = sum(d[0] for d in data); tot_s = sum(d[1] for d in data) or 1
print(sec[0][:120]); print(f"total warp-instr {tot_i:.3e}  samples {tot_s}")
for d in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"{d[1]/tot_s*100:5.1f}% {d[0]:>11} thr {d[2]:4.1f} {d[3]} {d[4][:80]}")
