"""K1 per-CTA device timeline (scratch build with -DESS_K1_PROF): entry, setup done,
first accumulator ready (epilogue), epilogue done, exit — relative to the earliest
entry, beside the event-timed launch.  k1_phases.py LIB  (env SHAPES="B:L,...")."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2512_10576_b200.decode import _e4m3  # noqa: E402
from paper_2512_10576_b200.indexer import indexer_logits  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for t in os.environ.get("SHAPES", "1:32768,4:32768,16:32768").split(","):
    B, L = (int(x) for x in t.split(":"))
    g = torch.Generator(device="cuda").manual_seed(0)
    k = _e4m3(torch.randn((B, L, 128), device="cuda", generator=g) * 8)
    ks = torch.rand((B, L), device="cuda", generator=g) + 0.5
    q = _e4m3(torch.randn((B, 64, 128), device="cuda", generator=g) * 4)
    w = torch.randn((B, 64), device="cuda", generator=g) / 8
    lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
    out = torch.empty((B, L), device="cuda")
    for _ in range(3):
        indexer_logits(q, w, k, ks, lens, out=out)
    flush.fill_(1)
    torch.cuda.synchronize()
    _lib.load().ess_debug_k1_prof_reset()
    torch.cuda._sleep(1_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); indexer_logits(q, w, k, ks, lens, out=out); b.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * 6))()
    _lib.load().ess_debug_k1_prof(buf)
    p = np.frombuffer(buf, dtype=np.uint64).reshape(160, 6)[:148, :5].astype(np.int64)
    p = (p - p[:, 0].min()) / 1e3
    print(f"B={B} L={L}: event {a.elapsed_time(b) * 1e3:.1f} us; span entry->last exit {p[:, 4].max():.1f} us")
    for i, nm in enumerate(["entry", "setup", "first acc", "epi done", "exit"]):
        print(f"  {nm:10s} min {p[:, i].min():6.2f}  med {np.median(p[:, i]):6.2f}  max {p[:, i].max():6.2f}")
