"""Device timeline of the CAPTURED decode step (the graph bench.py replays): every
stage of DSADecodeLayer.attend is followed by an ess_timestamp node on the stream it
ran on, so the graph records where each stage ended (globaltimer, ns).  The stamp
nodes perturb the step: besides ~1-2 us each on the chain, they slow the first K1 from
~17 us (scripts/k1_in_graph.py, no stamps) to ~27 us.  Read order and shares, not
absolutes.
Env: CONFIG=c2|c3|c4, STEPS, K1PROF=1 (with ESS_LIB = a -DESS_K1_PROF build),
B2B=n (n back-to-back replays per printed step)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib, decode  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows  # noqa: E402

CFG = {"c2": (64, 32768, 0.25), "c4": (64, 131072, 0.1),
       "c3": (16, 32768, 0.25)}[os.environ.get("CONFIG", "c2")]  # c3: one layer of C3
B, ctx, rho = CFG
K1PROF = bool(os.environ.get("K1PROF"))  # with ESS_LIB=<a -DESS_K1_PROF build>
B2B = int(os.environ.get("B2B", 1))
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=96, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
stamps = torch.zeros(64, dtype=torch.int64, device="cuda")
names = []


def mark(name):
    i = len(names)
    names.append(name)
    _lib.check(_lib.load().ess_timestamp(stamps[i:].data_ptr(), _lib.stream_handle()), "ts")


def wrap(mod, fn_name, label):
    f = getattr(mod, fn_name)

    def g(*a, **k):
        r = f(*a, **k)
        mark(label)
        return r
    setattr(mod, fn_name, g)


wrap(decode, "indexer_logits", "K1 indexer")
wrap(decode, "topk", "K2 topk")
wrap(decode, "topk_split", "K2+K3a topk+split")
wrap(decode, "gather", "K4 gather (side)")
wrap(decode, "sparse_mla_da", "K5 fused DA")
wrap(decode, "sparse_mla", "K5 pass")
wrap(decode, "indexer_logits_stream", "K1 stream")
wrap(decode, "topk_split_stream", "K2+K3a stream")
wrap(decode, "gather_stream", "K4 stream (side)")
acc_f = decode.PoolSet.access


def access(self, *a, **k):
    r = acc_f(self, *a, **k)
    mark("K3(b) LRU")
    return r


decode.PoolSet.access = access
split_f, settle_f = decode.PoolSet.split, decode.PoolSet.settle


def split(self, *a, **k):
    r = split_f(self, *a, **k)
    mark("K3a split")
    return r


def settle(self, *a, **k):
    r = settle_f(self, *a, **k)
    mark("settle")
    return r


decode.PoolSet.split, decode.PoolSet.settle = split, settle
adm_f = DSADecodeLayer._append_device


def append_dev(self, *a, **k):
    r = adm_f(self, *a, **k)
    mark("admit")
    return r


DSADecodeLayer._append_device = append_dev
dev_step = DSADecodeLayer._device_step


def device_step(self, *a, **k):
    mark("start")
    dev_step(self, *a, **k)
    mark("end")


DSADecodeLayer._device_step = device_step
layer.micro = int(os.environ.get("MICRO", 2))
layer.first_frac = float(os.environ["FIRST"]) if os.environ.get("FIRST") else None
layer.attend(*layer.next_queries(), overlap=os.environ.get("OVERLAP", "dba"), micro=layer.micro)
layer.append_token()  # one eager step: the deferred-settle state of the steady step
torch.cuda.synchronize()
names.clear()
layer.first_frac = float(os.environ["FIRST"]) if os.environ.get("FIRST") else None
layer.capture(os.environ.get("OVERLAP", "dba"), 32)  # eager step (stamps 0..n-1), then the graph (stamps n..2n-1)
n = len(names) // 2
gnames = names[n:]
steps = int(os.environ.get("STEPS", 6))
for t in range(steps):
    q_idx, q = layer.next_queries()
    rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
    torch.cuda.synchronize()
    if K1PROF:
        _lib.load().ess_debug_k1_prof_reset()
    for _ in range(B2B):  # back-to-back replays (no host gap): the last one is read
        layer.step(q_idx, q, rows)
    torch.cuda.synchronize()
    if t >= steps - 3:
        s = stamps.cpu().tolist()[n:2 * n]
        if K1PROF:  # scratch -DESS_K1_PROF lib: the first K1 launch's CTAs in the graph
            buf = (ctypes.c_ulonglong * (160 * 6))()
            _lib.load().ess_debug_k1_prof(buf)
            p = np.frombuffer(buf, dtype=np.uint64).reshape(160, 6)[:148, :5].astype(np.int64)
            live = p[:, 0] > 0
            p = (p[live] - s[0]) / 1e3
            print("  K1[0] vs start: " + "  ".join(
                f"{nm} {p[:, i].min():.1f}/{np.median(p[:, i]):.1f}/{p[:, i].max():.1f}"
                for i, nm in enumerate(["entry", "setup", "first-acc", "epi-done", "exit"])))
        m = int(layer.step_counts()[:, 1].sum())
        print(f"step {t}: misses {m}  " + "  ".join(f"{nm}={(s[i] - s[0]) / 1e3:.1f}"
                                                  for i, nm in enumerate(gnames) if i))
