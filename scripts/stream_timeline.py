"""Per-request timeline of the streamed step (overlap="stream") from a -DESS_STREAM_PROF
scratch library (ESS_LIB=scratch_libs/sprof.so, built by scripts/variant_lib.sh over
topk.cu AND pool.cu): for each request, when its top-k started (its logits complete),
when its split was published and when its last miss row landed, relative to the
step's first top-k start; plus the step's graph time."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

B, ctx, rho = {"c2": (64, 32768, 0.25), "c4": (64, 131072, 0.1)}[os.environ.get("CONFIG", "c2")]
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=64, seed=1234, drift=0.97)
if os.environ.get("MICRO"):
    layer.micro = int(os.environ["MICRO"])
if os.environ.get("FIRST"):
    layer.first_frac = float(os.environ["FIRST"])
layer.prefill_warmup(windows=32)
L = _lib.load()
for fn in (L.ess_debug_stream_prof_topk, L.ess_debug_stream_prof_gather, L.ess_debug_stream_prof_k1):
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * (1024 * 4))()
buf2 = (ctypes.c_ulonglong * (1024 * 4))()
buf3 = (ctypes.c_ulonglong * (1024 * 4))()
OV = os.environ.get("OVERLAP", "stream")
layer.capture(OV, 32)
for t in range(6):
    q_idx, q = layer.next_queries()
    rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
    torch.cuda.synchronize()
    L.ess_debug_stream_prof_topk(None, 1)
    L.ess_debug_stream_prof_gather(None, 1)
    L.ess_debug_stream_prof_k1(None, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stamp = torch.zeros(2, dtype=torch.int64, device="cuda")
    e0.record()
    _lib.check(L.ess_timestamp(stamp[0:].data_ptr(), _lib.stream_handle()), "ts")
    layer.step(q_idx, q, rows)
    _lib.check(L.ess_timestamp(stamp[1:].data_ptr(), _lib.stream_handle()), "ts")
    e1.record()
    torch.cuda.synchronize()
    L.ess_debug_stream_prof_topk(buf, 0)
    L.ess_debug_stream_prof_gather(buf2, 0)
    L.ess_debug_stream_prof_k1(buf3, 0)
    k1 = np.frombuffer(buf3, dtype=np.uint64).reshape(1024, 4)
    p = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 4)[:B, :3].astype(np.int64)
    p[:, 2] = np.frombuffer(buf2, dtype=np.uint64).reshape(1024, 4)[:B, 2].astype(np.int64)
    st = stamp.cpu().tolist()
    t0 = st[0]
    rel = (p - t0) / 1e3
    m = layer.step_counts()[:, 1].cpu().numpy()
    if t >= 3:
        print(f"step {t}: graph {e0.elapsed_time(e1) * 1e3:.1f} us, end stamp {(st[1] - t0) / 1e3:.1f}, "
              f"misses {m.sum()} (times from the stamp before the graph launch)")
        for b in list(range(0, B, 8)) + [B - 1]:
            print(f"  req {b:2d}: logits {(int(k1[b, 3]) - t0) / 1e3:6.1f}  topk {rel[b, 0]:6.1f}  ready {rel[b, 1]:6.1f}  landed {rel[b, 2]:6.1f}  (misses {m[b]})")
        print(f"  last landed {rel[:, 2].max():.1f}; ready span {rel[:, 1].min():.1f}..{rel[:, 1].max():.1f}")
        order = np.argsort(rel[:, 2])
        land = rel[order, 2]
        cum = np.cumsum(m[order]) * 704 / 1e3  # KB landed
        for f in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
            i = min(len(land) - 1, int(f * len(land)) - (1 if f == 1.0 else 0))
            print(f"    {f:4.2f} of requests landed by {land[i]:6.1f} us ({cum[i] / 1e3:.2f} MB)")
