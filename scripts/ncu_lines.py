"""Warp-stall samples aggregated per CUDA source line (file:line) from an ncu report:
ncu_lines.py REP KERNEL_REGEX [N].  Uses the interleaved cuda,sass source page."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
agg, text = defaultdict(float), {}
fname, line = "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0].isdigit():  # a source line row: Line No, Source, Address, Source, samples...
        line = (fname, int(r[0]))
        text[line] = r[1].strip()[:80]
        if len(r) > 4 and r[4]:
            try:
                agg[line] += float(r[4])
            except ValueError:
                pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]:<5} {text.get(k, '')}")
