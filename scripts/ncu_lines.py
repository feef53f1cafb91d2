"""Per CUDA source line of one kernel (ncu source page, cuda+sass view): warp
instructions executed and stall samples, top N. usage: ncu_lines.py REPORT KERNEL [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout.splitlines()
rows, f = [], "?"
for r in csv.reader(out):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] and r[0] != "Line No" and r[0].isdigit():
        try:
            rows.append((int(r[7]) if r[7] not in ("-", "") else 0, int(r[4]) if r[4] not in ("-", "") else 0,
                         f"{f}:{r[0]}", r[1].strip()))
        except (ValueError, IndexError):
            pass
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"instructions {ti:.3e}  samples {ts}")
for x in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{x[0]/ti*100:5.1f}% instr {x[1]/ts*100:5.1f}% stall  {x[2]:<22} {x[3][:90]}")
