"""K4 alone on REAL miss lists: a C2/C4 decode layer after warm-up, one product step,
then the gather of that step's misses re-timed at several CTA counts (idempotent)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402
from paper_2512_10576_b200.transfer import gather  # noqa: E402

B, ctx, rho = {"c2": (64, 32768, 0.25), "c4": (64, 131072, 0.1)}[os.environ.get("CONFIG", "c4")]
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=16, seed=1234, drift=0.97,
                       hugepages=os.environ.get("HP", "1") == "1")
layer.prefill_warmup(windows=32)
for _ in range(3):
    layer.attend(*layer.next_queries(), overlap="none")
    layer.append_token()
acc = layer.acc
m = acc.counts[:, 1].cpu()
ids = acc.miss_ids.cpu()
gaps = []
for b in range(4):
    v = ids[b, :int(m[b])].sort().values
    gaps.append((v[1:] - v[:-1] == 1).float().mean().item() if len(v) > 1 else 0)
byt = int(m.sum()) * 656
print(f"store {layer.store.nbytes / 2**30:.1f} GiB hugepages={layer.store.hugepages}; misses/req {m.float().mean():.1f}; "
      f"adjacent-id fraction {sum(gaps) / len(gaps):.2f}")
for ctas in (20, 32, 64, 148):
    for bulk in (False, True):
        for _ in range(2):
            gather(layer.pool, layer.store, acc, max_ctas=ctas, bulk=bulk)
        ts = []
        for _ in range(7):
            torch.cuda.synchronize()
            torch.cuda._sleep(1_000_000)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gather(layer.pool, layer.store, acc, max_ctas=ctas, bulk=bulk); e.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
        ts.sort()
        print(f"{'bulk' if bulk else 'ld16'} ctas={ctas}: {ts[3]:.1f} us {byt / ts[3] / 1e3:.1f} GB/s")
