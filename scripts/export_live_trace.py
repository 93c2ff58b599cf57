"""Run the product decode step at the C1 shape (B=4, ctx 4K, rho 0.25, 2048 of 4K) for a
few steps with the live selection recorder on, and write request 0's ESSTRACE plus
the device cache manager's per-step miss counts (the fixture tests/golden/live_c1.*
is this script's output)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer, SelectionRecorder  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/live_c1"
B, ctx, rho, steps = 4, 4096, 0.25, int(os.environ.get("STEPS", 12))
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=steps + 4, seed=7, drift=0.97)
rec = SelectionRecorder([layer])
rec.prefill([layer.prefill_warmup(windows=8, record=True)])
misses = []
for _ in range(steps):
    layer.attend(*layer.next_queries())
    torch.cuda.synchronize()
    rec.record()
    misses.append(layer.step_counts()[:, 1].tolist())
    layer.append_token()
layer.pool.check()
rec.write(0, out + ".esstrace")
with open(out + ".json", "w") as f:
    json.dump({"config": "C1: B=4, ctx 4096, rho 0.25, top-k 2048, 8 prefill windows, drift 0.97",
               "request": 0, "sparse_ratio": rho,
               "device_misses_per_step": [m[0] for m in misses]}, f, indent=1)
print("wrote", out + ".esstrace", [m[0] for m in misses])
