"""Aggregate an ncu source page (cuda view) of one kernel over named line ranges of
one file: warp instructions and stall samples per range. Lines of other files
(inlined helpers) are attributed to '<file>'.
usage: ncu_ranges.py REPORT KERNEL[@FUNCSUBSTR] FILE name:a-b [name:a-b ...]
(@FUNCSUBSTR picks one instantiation, e.g. k_pass_x64@"(int)1,")"""
import csv, subprocess, sys
rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
kern, _, fsub = kern.partition("@")
ranges = []
for s in sys.argv[4:]:
    n, ab = s.split(":")
    a, b = ab.split("-")
    ranges.append((n, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout.splitlines()
agg, f, fn = {}, "?", ""
for r in csv.reader(out):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] == "Function Name":
        fn = r[1]
    elif r and r[0].isdigit() and fsub in fn:
        try:
            ins = int(r[7]) if r[7] not in ("-", "") else 0
            smp = int(r[4]) if r[4] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        ln = int(r[0])
        key = f"<{f}>"
        if f == fname:
            key = next((n for n, a, b in ranges if a <= ln <= b), f"{fname}:other")
        a = agg.setdefault(key, [0, 0])
        a[0] += ins
        a[1] += smp
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti:.3e}  samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:<24} instr {v[0]/ti*100:5.1f}%  stall-samples {v[1]/ts*100:5.1f}%")
