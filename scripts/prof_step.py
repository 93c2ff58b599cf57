"""Minimal C2 decode-step driver for ncu (no CPU leg, no ceiling, no e2e).

    ncu --set full -k regex:sparse_mla -s 2 -c 1 -o gpurun_out/prof python scripts/prof_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--rho", type=float, default=0.25)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--windows", type=int, default=4)
ap.add_argument("--overlap", default="da")
a = ap.parse_args()
layer = DSADecodeLayer(a.batch, a.ctx, a.rho, 2048, max_new_tokens=a.steps + 8, seed=5, drift=0.97)
layer.prefill_warmup(windows=a.windows)
for _ in range(a.steps):
    q_idx, q = layer.next_queries()
    layer.attend(q_idx, q, overlap=a.overlap)
    layer.append_token()
torch.cuda.synchronize()
layer.pool.check()
print("prof_step done")
