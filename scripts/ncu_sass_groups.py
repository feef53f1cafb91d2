"""Hot SASS regions of one kernel instantiation from an ncu report: consecutive
instructions with equal execution counts are grouped; prints the share of warp
instructions, the average active threads per warp and the first instruction.
usage: ncu_sass_groups.py REPORT KERNEL_REGEX NAME_SUBSTR [MIN_SHARE]"""
import csv, subprocess, sys
rep, kern, sub = sys.argv[1], sys.argv[2], sys.argv[3]
mn = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        secs.append(cur)
    elif cur is not None:
        cur[1].append(r)
name, rs = next((n, r) for n, r in secs if sub in n)
h = next(r for r in rs if r and r[0] == "Address")
A, S, IE, TE, SMP = (h.index(k) for k in ("Address", "Source", "Instructions Executed", "Thread Instructions Executed",
                                          "Warp Stall Sampling (All Samples)"))
data = []
for r in rs:
    try:
        data.append((int(r[A], 16), r[S], int(r[IE] or 0), int(r[TE] or 0), int(r[SMP] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data) or 1
tt = sum(d[3] for d in data)
ts = sum(d[4] for d in data) or 1
print(name[:90])
print(f"warp-instr {tot:.3e}  avg threads/instr {tt / tot:.1f}")
grp = []
for d in data:
    if grp and grp[-1][1] == d[2]:
        g = grp[-1]
        g[2] += 1; g[3] += d[3]; g[4] += d[4]
    else:
        grp.append([d[0], d[2], 1, d[3], d[4], d[1]])
for g in grp:
    if g[1] * g[2] > mn * tot:
        print(f"{hex(g[0])[-5:]} x{g[1] / 1e6:8.2f}M n={g[2]:4d} instr {g[1] * g[2] / tot * 100:5.1f}% "
              f"stall {g[4] / ts * 100:5.1f}% thr {g[3] / max(g[1] * g[2], 1):5.1f}  {g[5].strip()[:50]}")
