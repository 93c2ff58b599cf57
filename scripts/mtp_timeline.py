"""Device timeline of the captured MTP step (MTPDecodeLayer, C2 shapes, MTP = 2): a
timestamp node after every stage on the stream it ran on (end times in us from the
step's first node).  Stamps perturb the step; read order and shares."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib, mtp  # noqa: E402
from paper_2512_10576_b200.decode import random_latent_rows  # noqa: E402

B, ctx, rho = 64, 32768, 0.25
layer = mtp.MTPDecodeLayer(B, ctx, rho, 2048, mtp=2, max_new_tokens=32, seed=4321, drift=0.97)
layer.micro = int(os.environ.get("MICRO", 2))
layer.first_frac = float(os.environ.get("FIRST", 0.25))
layer.prefill_warmup(windows=32)
stamps = torch.zeros(64, dtype=torch.int64, device="cuda")
names = []


def mark(name):
    i = len(names)
    names.append(name)
    _lib.check(_lib.load().ess_timestamp(stamps[i:].data_ptr(), _lib.stream_handle()), "ts")


def wrap(mod, fn, label):
    f = getattr(mod, fn)

    def g(*a, **k):
        r = f(*a, **k)
        mark(label if fn != "sparse_mla" else f"{label} {k.get('mode', 'full')}")
        return r
    setattr(mod, fn, g)


for fn, label in (("indexer_logits_mtp", "K1"), ("topk_mtp", "K2"), ("gather", "K4"), ("sparse_mla", "K5")):
    wrap(mtp, fn, label)
acc_f = mtp.MTPDecodeLayer.__mro__[1].__dict__  # noqa: F841
pa = mtp.AccessBatch  # noqa: F841
from paper_2512_10576_b200.cache import PoolSet  # noqa: E402
am = PoolSet.access_mtp


def access_mtp(self, *a, **k):
    r = am(self, *a, **k)
    mark("K3")
    return r


PoolSet.access_mtp = access_mtp
ds = mtp.MTPDecodeLayer._device_step


def device_step(self, *a, **k):
    mark("start")
    ds(self, *a, **k)
    mark("end")


mtp.MTPDecodeLayer._device_step = device_step
ov = os.environ.get("OVERLAP", "dba")
layer.capture(ov, 32)
n = len(names) // 2
gn = names[n:]
rng = np.random.default_rng(0)
for t in range(5):
    acc = mtp.draw_accepted(rng, B, 1.7, 3)
    q_idx, q = layer.next_queries(acc)
    rows = random_latent_rows(B * 3, "cuda", layer.gen).view(B, 3, 656)
    layer.step(q_idx, q, rows, torch.from_numpy(acc).cuda(), max_accepted=int(acc.max()))
    torch.cuda.synchronize()
    if t >= 3:
        s = stamps.cpu().tolist()[n:2 * n]
        print(f"step {t}: " + "  ".join(f"{nm}={(s[i] - s[0]) / 1e3:.1f}" for i, nm in enumerate(gn) if i))
