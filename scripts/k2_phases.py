"""K2 per-phase device time (scratch build with -DESS_TOPK_PROF) on real C2 logits."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402
from paper_2512_10576_b200.indexer import indexer_logits, topk  # noqa: E402

B, ctx = 64, int(os.environ.get("CTX", 32768))
layer = DSADecodeLayer(B, ctx, 0.25, 2048, max_new_tokens=16, seed=1234, drift=0.97)
q_idx, q = layer.next_queries()
indexer_logits(q_idx, layer.w, layer.k_cache, layer.k_scale, layer.lens, out=layer.logits)
for _ in range(2):
    topk(layer.logits, layer.lens, layer.K, out=layer.idx, count=layer.cnt)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (1024 * 12))()
_lib.load().ess_debug_topk_prof(buf)
full = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 12)[:B].astype(np.int64)
a = full[:, :7]
d = np.diff(a, axis=1) / 1e3
names = ["stage+hist12", "pick d1", "list compact", "2x10-bit digits", "counts", "emit"]
for i, nm in enumerate(names):
    print(f"{nm:18s} mean {d[:, i].mean():6.2f} us  max {d[:, i].max():6.2f}")
print(f"total mean {(a[:, 6] - a[:, 0]).mean() / 1e3:.2f} us; span {(a[:, 6].max() - a[:, 0].min()) / 1e3:.2f} us")
print("list sizes m (first 8 rows):", [int(x) for x in full[:8, 7]])
print(f"list: pass1 {((full[:, 8] - full[:, 2]) / 1e3).mean():.2f} us, scan {((full[:, 9] - full[:, 8]) / 1e3).mean():.2f} us, "
      f"pass2 {((full[:, 3] - full[:, 9]) / 1e3).mean():.2f} us")
