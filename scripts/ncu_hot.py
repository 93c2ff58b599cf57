"""Top SASS lines by warp-stall samples from an ncu report: ncu_hot.py REP KERNEL_REGEX [N]."""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, ci = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) <= ci or not r[0].startswith("0x"):
        continue
    data.append((float(r[ci] or 0), r[0][-5:], r[si].strip()))
tot = sum(d[0] for d in data) or 1
for a, addr, s in sorted(data, reverse=True)[:n]:
    print(f"{a / tot * 100:5.1f}% {addr} {s}")
