"""K3 per-phase device time (scratch build with -DESS_POOL_PROF): C2 layer, one access."""
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

B, ctx, rho = 64, 32768, 0.25
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=16, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
for _ in range(3):
    layer.attend(*layer.next_queries(), overlap="none")
    layer.append_token()
q_idx, q = layer.next_queries()
indexer_logits(q_idx, layer.w, layer.k_cache, layer.k_scale, layer.lens, out=layer.logits)
topk(layer.logits, layer.lens, layer.K, out=layer.idx, count=layer.cnt)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
torch.cuda.synchronize()
layer.pool.access(layer.idx, layer.cnt, out=layer.acc)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 16))()
_lib.load().ess_debug_pool_prof(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 16)[:B, :8].astype(np.int64)
d = np.diff(a, axis=1) / 1e3
names = ["load+validate", "hit/miss split", "warmup-part/restamp", "select", "compaction", "victims+assign", "outputs"]
print("misses/req", float(layer.acc.counts[:, 1].float().mean()))
for i, nm in enumerate(names):
    print(f"{nm:22s} mean {d[:, i].mean():6.2f} us  max {d[:, i].max():6.2f}")
print(f"total (first stamp -> last) mean {(a[:, 7] - a[:, 0]).mean() / 1e3:.2f} us; "
      f"span over CTAs {(a[:, 7].max() - a[:, 0].min()) / 1e3:.2f} us")
sel = d[:, 3]
print("select per CTA (us):", " ".join(f"{x:.1f}" for x in sel))
c = layer.pool.counters().cpu().numpy()
print("cap/size:", c[:8, 0].tolist(), c[:8, 1].tolist())
full = np.frombuffer(buf, dtype=np.uint64).reshape(256, 16)[:B].astype(np.int64)
print("key min/max/range of slow CTAs:", [(i, int(full[i, 8]), int(full[i, 9]), int(full[i, 9] - full[i, 8])) for i in range(B) if sel[i] > 6])
print("typical:", [(i, int(full[i, 8]), int(full[i, 9]), int(full[i, 9] - full[i, 8])) for i in range(3)])
