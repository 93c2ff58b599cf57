"""Graph-captured step vs oracle, per overlap schedule (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import dsa  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

for overlap in ("none", "da"):
    B = 4
    layer = DSADecodeLayer(B, 8192, 0.25, 2048, max_new_tokens=12, seed=3, drift=0.97)
    layer.prefill_warmup(windows=6)
    layer.capture(overlap=overlap)
    for step in range(3):
        q_idx, q = layer.next_queries()
        rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
        hist = int(layer.lens[0])
        layer.step(q_idx, q, rows)
        torch.cuda.synchronize()
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        host = layer.store.host.numpy()
        c = layer.step_counts().cpu().numpy()
        errs = []
        for b in range(B):
            want = idx[b, :cnt[b]]
            ref_o, _ = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], layer.sm_scale)
            o = layer.out[b].float().cpu().numpy()
            errs.append(float(np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o)))
        print(overlap, "step", step, "hist", hist, "counts", c[:, :2].tolist(), "rel", [f"{e:.3g}" for e in errs])
        if overlap == "da":
            ws = layer._ws
            print("  ws_ml sample", ws.ml[0, :2].tolist())
    layer.close()
