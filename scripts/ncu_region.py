"""Print the SASS of one kernel whose execution count equals COUNT (a loop body)."""
import csv, subprocess, sys
rep, kern, count = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
sections, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]; sections.append(cur)
    elif cur is not None:
        cur.append(line)
sec = next(s for s in sections if kern in s[0])
rows = list(csv.reader(sec[1:])); h = rows[0]
IE, S, A, SMP = h.index("Instructions Executed"), h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
for r in rows[1:]:
    try:
        if int(r[IE] or 0) == count:
            print(r[A][-5:], f"{int(r[SMP] or 0):6d}", r[S].strip()[:100])
    except (ValueError, IndexError):
        pass
