"""Measure the B200 kernels on the reference's cost-table grid and write
profiles/b200_cost_table.csv (+ .transfer.json with the measured gather rate):

    python scripts/export_cost_table.py [--gather-gbs G] [--out PATH]

Feed it to the reference simulator: offsim simulate --profile profiles/b200_cost_table_full.csv
(see INTEGRATION.md §3 for the merge with a base profile for the ops outside the path)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10576_b200 import costbridge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "profiles", "b200_cost_table.csv"))
ap.add_argument("--gather-gbs", type=float, default=None)
a = ap.parse_args()
entries = costbridge.export(a.out, gather_gbs=a.gather_gbs)
for op, pts in entries.items():
    print(op, " ".join(f"({b:g},{c:g})={t:.1f}us" for b, c, t in pts))
print("->", a.out)
