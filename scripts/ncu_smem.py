"""Top shared-memory instructions of one kernel in an ncu source page: wavefronts,
excess (bank-conflict) wavefronts and stall samples. usage: ncu_smem.py REPORT KERNEL [TOP]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
c = {k: h.index(k) for k in ("Address", "Source", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
                              "Warp Stall Sampling (All Samples)", "Instructions Executed")}
def num(r, k):
    try:
        return float(r[c[k]] or 0)
    except ValueError:
        return 0.0
data = [r for r in rows[1:] if len(r) > max(c.values())]
tw = sum(num(r, "L1 Wavefronts Shared") for r in data) or 1
te = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
ts = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
print(f"shared wavefronts {tw:.3e}, excessive {te:.3e} ({te/tw*100:.1f}%), samples {ts:.0f}")
for r in sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared"))[:top]:
    print(f"{num(r,'L1 Wavefronts Shared')/tw*100:5.1f}% wf  exc {num(r,'L1 Wavefronts Shared Excessive')/tw*100:5.1f}%  "
          f"stall {num(r,'Warp Stall Sampling (All Samples)')/ts*100:4.1f}%  {r[c['Address']][-5:]} {r[c['Source']].strip()[:70]}")
