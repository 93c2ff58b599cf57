"""FP8 K5 (CTA pair) per-tile event times of request 0 (scratch build -DESS_MLA2_TRACE)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2512_10576_b200.attention import sparse_mla  # noqa: E402
from paper_2512_10576_b200.cache import PoolSet  # noqa: E402
from paper_2512_10576_b200.decode import random_latent_rows  # noqa: E402

B, cap, n = int(os.environ.get("B", 64)), 8192, 2048
FMT = int(os.environ.get("FMT", "656"))
pools = PoolSet(B, 32768, cap, cap, row_bytes=FMT)
g = torch.Generator(device="cuda").manual_seed(0)
rv = pools.rows_view()
for b in range(B):
    if FMT == 656:
        rv[b].copy_(random_latent_rows(cap, "cuda", g))
    else:
        rv[b].copy_((torch.randn(rv[b].shape, device="cuda", generator=g) * 0.5).half())
sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:n] for _ in range(B)]).int()
cnt = torch.full((B,), n, dtype=torch.int32, device="cuda")
q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
for _ in range(3):
    sparse_mla(pools, q, sel, cnt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sparse_mla(pools, q, sel, cnt); e1.record(); torch.cuda.synchronize()
print(f"launch {e0.elapsed_time(e1) * 1e3:.1f} us")
buf = (ctypes.c_ulonglong * (2 * 10 * 72))()
_lib.load().ess_debug_mla2_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 10, 72)[:, :, :64].astype(np.int64)
t0 = a[:, 0, 0].min()
names = ["ld issue", "stg full", "S deq", "V deq", "smx sees S", "P arrive", "mma S wait", "mma P seen", "mma V seen", "ld issued"]
for i in list(range(0, 5)) + list(range(30, 33)) + list(range(60, 64)):
    for r in (0, 1):
        ev = list(range(9)) + [9] if r == 0 else [0, 9, 1, 2, 3, 4, 5]
        print(f"tile {i:2d} r{r}: " + " ".join(f"{names[e]}={(a[r, e, i] - t0) / 1e3:6.2f}" for e in ev))
for r in (0, 1):
    for e in range(9 if r == 0 else 6):
        d = np.diff(a[r, e, 8:60]) / 1e3
        print(f"r{r} {names[e]:>12s}: period {d.mean():.3f} us")
for r in (0, 1):
    for e0_, e1_ in [(0, 9), (9, 1), (1, 2), (2, 3), (4, 5)]:
        print(f"r{r} {names[e0_]} -> {names[e1_]}: {((a[r, e1_, 8:60] - a[r, e0_, 8:60]) / 1e3).mean():.3f} us")
print(f"S deq (max r) -> mma S wait: {((a[0, 6, 8:60] - np.maximum(a[0, 2, 8:60], a[1, 2, 8:60])) / 1e3).mean():.3f} us")
print(f"mma S wait(i) -> smx sees S(i): {((a[0, 4, 8:60] - a[0, 6, 8:60]) / 1e3).mean():.3f} us")
print(f"P arrive (max r) -> mma P seen: {((a[0, 7, 8:60] - np.maximum(a[0, 5, 8:60], a[1, 5, 8:60])) / 1e3).mean():.3f} us")
print(f"ld issue(i) - V deq(i-3) [ring gate]: {((a[0, 0, 8:60] - a[0, 3, 5:57]) / 1e3).mean():.3f} us")
