"""K1 of the first micro-batch inside the captured C2 step (no timestamp nodes):
per-CTA entry -> epilogue done, from a -DESS_K1_PROF -DESS_K1_PROF_FULLGRID build.
k1_in_graph.py LIB   (env MB_FIRST: first micro-batch share)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ESS_LIB"] = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

B, ctx, rho = 64, 32768, 0.25
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=96, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
layer.micro, layer.first_frac = 2, float(os.environ.get("MB_FIRST", 0.25))
layer.capture("dba", 32)
L = _lib.load()
for t in range(6):
    q_idx, q = layer.next_queries()
    rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    layer.step(q_idx, q, rows)
    b.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * 6))()
    L.ess_debug_k1_prof(buf)
    p = np.frombuffer(buf, dtype=np.uint64).reshape(160, 6)[:148, :5].astype(np.int64)
    p = (p - p[:, 0].min()) / 1e3
    print(f"step {t}: {a.elapsed_time(b) * 1e3:.0f} us (incl. input copies); K1[0] first-acc med "
          f"{np.median(p[:, 2]):.1f}  epi-done med {np.median(p[:, 3]):.1f} max {p[:, 3].max():.1f}"
          f"  exit max {p[:, 4].max():.1f}", flush=True)
