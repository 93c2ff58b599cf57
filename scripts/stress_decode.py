"""Stress: many decode steps per schedule, attention checked against the oracle each
step; prints the failing (schedule, step, request) if any."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import dsa  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

STEPS = int(os.environ.get("STEPS", 30))
bad = 0
for mode in ("eager-none", "eager-da", "graph-da", "graph-none"):
    B = 6
    layer = DSADecodeLayer(B, 8192, 0.25, 2048, max_new_tokens=STEPS + 8, seed=11, drift=0.9)
    layer.prefill_warmup(windows=4)
    if mode.startswith("graph"):
        layer.capture(overlap=mode.split("-")[1])
    worst = 0.0
    for step in range(STEPS):
        q_idx, q = layer.next_queries()
        rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
        if mode.startswith("graph"):
            layer.step(q_idx, q, rows)
        else:
            layer.attend(q_idx, q, overlap=mode.split("-")[1])
            layer.append_token(new_rows=rows)
        torch.cuda.synchronize()
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        host = layer.store.host.numpy()
        for b in range(B):
            want = idx[b, :cnt[b]]
            ref_o, _ = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], layer.sm_scale)
            o = layer.out[b].float().cpu().numpy()
            e = float(np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o))
            worst = max(worst, e if np.isfinite(e) else 1e9)
            if not (e <= 1e-2):
                bad += 1
                c = layer.step_counts().cpu().numpy()[b]
                print(f"FAIL {mode} step {step} req {b} rel {e:.3g} counts {c.tolist()}")
    print(mode, "worst rel", worst)
    layer.close()
print("bad", bad)
