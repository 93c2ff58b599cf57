"""Per-step view of the e2e loop (layer.step_host at C2): host enqueue time and device
time of every step, to see whether e2e variance is a few slow steps or a slow link.
Env: STEPS."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

B, K = 64, int(os.environ.get("STEPS", 40))
layer = DSADecodeLayer(B, 32768, 0.25, 2048, max_new_tokens=2 * K + 32, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
layer.micro, layer.first_frac = 2, 0.25
layer.capture("dba", 32)
inputs = [layer.next_queries() for _ in range(K)]
rows = [random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656) for _ in range(K)]
h_in = [(a.cpu().pin_memory(), b.cpu().pin_memory()) for a, b in inputs]
h_out = [torch.empty(layer.out.shape, dtype=layer.out.dtype).pin_memory() for _ in range(K)]
for t in range(3):
    layer.step_host(h_in[t][0], h_in[t][1], rows[t], h_out[t])
layer.host_sync()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
host = []
ev[0].record()
for t in range(K):
    t0 = time.perf_counter()
    layer.step_host(h_in[t][0], h_in[t][1], rows[t], h_out[t])
    host.append((time.perf_counter() - t0) * 1e6)
    ev[t + 1].record()
layer._ds.synchronize()
end = torch.cuda.Event(enable_timing=True)
end.record()
torch.cuda.synchronize()
dev = [ev[t].elapsed_time(ev[t + 1]) * 1e3 for t in range(K)]
tot = ev[0].elapsed_time(end) * 1e3
print(f"total {tot / K:.0f} us/step -> {B * K / tot * 1e6:.0f} tok/s; host enqueue med "
      f"{sorted(host)[K // 2]:.0f} max {max(host):.0f} us")
print("device us per step:", " ".join(f"{x:.0f}" for x in dev))
