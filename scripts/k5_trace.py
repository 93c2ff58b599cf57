"""K5 per-tile event times of CTA (0,0) (scratch build with -DESS_MLA_TRACE) at C2 shape."""
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

B, cap, n = int(os.environ.get("B", 64)), 8192, 2048
pools = PoolSet(B, 32768, cap, cap, row_bytes=1152)
g = torch.Generator(device="cuda").manual_seed(0)
rv = pools.rows_view()
rv.copy_((torch.randn(rv.shape, device="cuda", generator=g) * 0.5).half())
sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:n] for _ in range(B)]).int()
cnt = torch.full((B,), n, dtype=torch.int32, device="cuda")
q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
for _ in range(3):
    sparse_mla(pools, q, sel, cnt)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 72))()
_lib.load().ess_debug_mla_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8, 72)[:6, :64].astype(np.int64)
t0 = a[0, 0]
names = ["rows in smem", "S issued", "softmax sees S", "P arrived", "MMA sees P", "PV issued"]
for i in list(range(0, 6)) + list(range(30, 34)) + list(range(60, 64)):
    print(f"tile {i:2d}: " + "  ".join(f"{nm}={(a[e, i] - t0) / 1e3:6.2f}" for e, nm in enumerate(names)))
d = np.diff(a[5, 8:60]) / 1e3
print(f"steady per-tile period (PV issue to PV issue): {d.mean():.3f} us")
for e in range(1, 6):
    print(f"  {names[e - 1]:>16s} -> {names[e]:<16s}: {((a[e, 8:60] - a[e - 1, 8:60]) / 1e3).mean():7.3f} us")
print(f"  S issued(i+1) - PV issued(i): {((a[1, 9:61] - a[5, 8:60]) / 1e3).mean():.3f} us")
