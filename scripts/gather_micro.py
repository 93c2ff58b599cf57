"""K4 zero-copy gather alone: B=64 pools, M misses each, sweep of CTA counts.
Also times a plain cudaMemcpy H2D of the same bytes for the link's DMA rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_10576_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])  # a scratch variant build
from paper_2512_10576_b200.cache import AccessBatch, PoolSet
from paper_2512_10576_b200.transfer import HostLatentStore, gather

B, cap, hist = 64, 8192, int(os.environ.get("HIST", 32768))
M = int(os.environ.get("M", 120))
pools = PoolSet(B, hist, cap, cap, row_bytes=int(os.environ.get("FMT", "1152")))
store = HostLatentStore(B, hist, hugepages=os.environ.get("HP", "1") == "1")
print(f"host store {store.nbytes / 2**30:.2f} GiB hugepages={store.hugepages} numa={store.numa_node}")
store.host.random_(0, 256)
g = torch.Generator(device="cuda").manual_seed(0)
K = 2048
z = lambda: torch.zeros((B, K), dtype=torch.int32, device="cuda")  # noqa: E731
acc = AccessBatch(counts=torch.zeros((B, 4), dtype=torch.int32, device="cuda"), sel_row=z(),
                  miss_ids=z(), miss_row=z(), hit_row=z())
acc.counts[:, 1] = M
for b in range(B):
    if os.environ.get("SEQ") == "1":  # contiguous host rows (page locality probe)
        acc.miss_ids[b, :M] = torch.arange(M, device="cuda", dtype=torch.int32) + 1000
    elif os.environ.get("SORTED") == "1":
        acc.miss_ids[b, :M] = torch.randperm(hist, device="cuda", generator=g)[:M].sort().values.int()
    else:
        acc.miss_ids[b, :M] = torch.randperm(hist, device="cuda", generator=g)[:M].int()
    acc.miss_row[b, :M] = torch.randperm(cap, device="cuda", generator=g)[:M].int()
byt = B * M * 656
for ctas in [int(c) for c in os.environ.get("CTAS", "8,20,40,80,148,296").split(",")]:
    for bulk in (False, True):
        for _ in range(3):
            gather(pools, store, acc, max_ctas=ctas, bulk=bulk)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gather(pools, store, acc, max_ctas=ctas, bulk=bulk); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        print(f"{'bulk' if bulk else 'ld16'} gather ctas={ctas:4d} M={M}: median {ts[5]:.1f} us  {byt / ts[5] / 1e3:.1f} GB/s")
hbuf = torch.empty(byt, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(byt, dtype=torch.uint8, device="cuda")
for _ in range(3):
    dbuf.copy_(hbuf, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); dbuf.copy_(hbuf, non_blocking=True); b.record(); torch.cuda.synchronize()
print(f"memcpy H2D {byt} B: {a.elapsed_time(b) * 1e3:.1f} us {byt / a.elapsed_time(b) / 1e6:.1f} GB/s")
