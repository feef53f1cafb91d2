"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: ncu_lines.py REPORT.ncu-rep KERNEL_DEMANGLED_SUBSTR MANGLED_SUBSTR [SO] [TOP]
Maps each SASS address of the profiled kernel (ncu --page source, sass) to its
source line via nvdisasm -gi on the cubin embedded in SO (innermost inlined line).
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

rep, kern, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
so = sys.argv[4] if len(sys.argv) > 4 else "paper_2602_19873_b200/libsfcnl_b200.so"
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
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
A, SMP, IE = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ins = []
for r in rows[1:]:
    try:
        ins.append((int(r[A], 16), int(r[SMP] or 0), int(r[IE] or 0)))
    except (ValueError, IndexError):
        pass
base = ins[0][0]

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
linemap = None
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    # the inline chain precedes an instruction innermost first; attribute to the
    # innermost frame outside the generic helpers (common.cuh) unless INNER=1
    inner = os.environ.get("INNER") == "1"
    fn, cur_line, pend, m = None, None, [], {}
    for L in dis.splitlines():
        t = L.strip()
        if t.startswith(".text.") and t.endswith(":"):
            fn = t[6:-1]
            cur_line, pend = None, []
            continue
        if fn is None or mangled not in fn:
            continue
        mm = re.match(r'//## File "([^"]+)", line (\d+)', t)
        if mm:
            pend.append((os.path.basename(mm.group(1)), int(mm.group(2))))
            continue
        mo = re.match(r"/\*([0-9a-f]{4,})\*/", t)
        if mo:
            if pend:
                pick = [fl for fl in pend if fl[0] != "common.cuh"] or pend
                cur_line = pend[0] if inner else pick[0]
                pend = []
            if cur_line:
                m[int(mo.group(1), 16)] = cur_line
    if m:
        linemap = m
        break
if not linemap:
    sys.exit("kernel not found in cubins: " + mangled)

agg = collections.defaultdict(lambda: [0, 0])
tot_s = sum(s for _, s, _ in ins) or 1
tot_i = sum(i for _, _, i in ins) or 1
for addr, s, ie in ins:
    key = linemap.get(addr - base, ("?", 0))
    agg[key][0] += s
    agg[key][1] += ie
src = {}
for (f, ln) in agg:
    if f != "?" and f not in src:
        p = glob.glob(f"paper_2602_19873_b200/csrc/{f}")
        src[f] = open(p[0]).read().splitlines() if p else []
print(f"{'file:line':28s} {'stall%':>7s} {'inst%':>6s}  source")
for (f, ln), (s, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    text = src.get(f, [])[ln - 1].strip()[:90] if f in src and 0 < ln <= len(src[f]) else ""
    print(f"{f + ':' + str(ln):28s} {100 * s / tot_s:7.2f} {100 * ie / tot_i:6.2f}  {text}")
