"""Feasibility: the batch as two independent half-batch layers whose captured steps
replay on two streams (two-batch overlap across steps) vs one full-batch layer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

CFG = {"c2": (64, 32768, 0.25), "c4": (64, 131072, 0.1)}[os.environ.get("CONFIG", "c2")]
B, ctx, rho = CFG
W, K = 5, 30
lanes = int(os.environ.get("LANES", 2))
overlap = os.environ.get("OVERLAP", "da")
micro = int(os.environ.get("MICRO", 1))
ls = []
for i in range(lanes):
    layer = DSADecodeLayer(B // lanes, ctx, rho, 2048, max_new_tokens=W + K + 16, seed=1234 + i, drift=0.97)
    layer.micro = micro
    layer.prefill_warmup(windows=32)
    ls.append(layer)
inputs = [[l.next_queries() for _ in range(W + K)] for l in ls]
rows = [random_latent_rows(B // lanes, "cuda").view(B // lanes, 1, 656) for _ in ls]
for l in ls:
    l.capture(overlap)
streams = [torch.cuda.Stream() for _ in ls]
cur = torch.cuda.current_stream()


def run(t0, t1):
    ev = torch.cuda.Event()
    ev.record(cur)
    for s in streams:
        s.wait_event(ev)
    for t in range(t0, t1):
        for i, (l, s) in enumerate(zip(ls, streams)):
            with torch.cuda.stream(s):
                l.step(inputs[i][t][0], inputs[i][t][1], rows[i])
    for s in streams:
        cur.wait_stream(s)


run(1, W)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
run(W, W + K)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / K
for l in ls:
    l.pool.check()
h = sum(l.access_totals()[0] for l in ls)
print(f"lanes={lanes} overlap={overlap} micro={micro}: {ms * 1e3:.1f} us/step {B / ms * 1e3:.0f} tok/s")
