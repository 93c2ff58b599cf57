"""Workloads for ncu captures of this round's kernels (one process per capture):
  mtp     C2 shapes, MTP = 2, eager steps (indexer_kernel<3>, topk rows, MTP access, K5 qtok)
  stream  C2, the streamed step eager (indexer_logits_stream, topk_stream_kernel,
          gather_stream_kernel)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

mode = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, ctx, rho = 64, 32768, 0.25
if mode == "mtp":
    from paper_2512_10576_b200.mtp import MTPDecodeLayer, draw_accepted
    layer = MTPDecodeLayer(B, ctx, rho, 2048, mtp=2, max_new_tokens=steps + 4, seed=4321, drift=0.97)
    layer.prefill_warmup(windows=32)
    rng = np.random.default_rng(0)
    for t in range(steps):
        acc = draw_accepted(rng, B, 1.7, 3)
        q_idx, q = layer.next_queries(acc)
        layer.attend(q_idx, q, overlap="dba")
        layer.append_tokens(acc)
else:
    from paper_2512_10576_b200.decode import DSADecodeLayer
    layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=steps + 4, seed=1234, drift=0.97)
    layer.prefill_warmup(windows=32)
    for t in range(steps):
        q_idx, q = layer.next_queries()
        layer.attend(q_idx, q, overlap="stream")
        layer.append_token()
torch.cuda.synchronize()
layer.pool.check(mode)
print(mode, "ok")
