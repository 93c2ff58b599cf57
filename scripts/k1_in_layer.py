"""K1 on the C2 layer's own buffers (micro-batch 0 slice), timed after a graph step,
back to back, and after an L2 flush — to split "K1 is slower inside the step" into
state left by the step (L2 / TLB) vs. concurrency.  k1_in_layer.py [K1PROF_LIB]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    os.environ["ESS_LIB"] = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402
from paper_2512_10576_b200.indexer import indexer_logits  # noqa: E402

B, ctx, rho = 64, 32768, 0.25
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=64, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
layer.micro, layer.first_frac = 2, 0.25
layer.capture("dba", 32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
prof = len(sys.argv) > 1
L = _lib.load()
n = int(os.environ.get("NREQ", 16))


def k1(tag):
    if prof:
        L.ess_debug_k1_prof_reset()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    indexer_logits(layer.q_idx_in[:n], layer.w[:n], layer.k_cache[:n], layer.k_scale[:n],
                   layer.lens[:n], out=layer.logits[:n])
    b.record()
    torch.cuda.synchronize()
    msg = f"{tag:28s} event {a.elapsed_time(b) * 1e3:6.1f} us"
    if prof:
        buf = (ctypes.c_ulonglong * (160 * 6))()
        L.ess_debug_k1_prof(buf)
        p = np.frombuffer(buf, dtype=np.uint64).reshape(160, 6)[:148, :5].astype(np.int64)
        p = (p - p[:, 0].min()) / 1e3
        msg += f"  first-acc med {np.median(p[:, 2]):.1f}  epi-done max {p[:, 3].max():.1f}"
    print(msg, flush=True)


for t in range(3):
    q_idx, q = layer.next_queries()
    rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
    layer.step(q_idx, q, rows)
    torch.cuda.synchronize()
    k1("after a graph step")
    k1("back to back")
    flush.fill_(1)
    torch.cuda.synchronize()
    k1("after a 256 MB L2 flush")
