"""K4 alone against the host store's size and backing (GPU page-table reach probe).

For each store (C2-sized 1.5 GB and C4-sized 5.9 GB at the 704-B pitch) and each backing
(ess_host_alloc with THP requested, without, and a cudaHostAlloc'd torch pinned buffer),
times the zero-copy gather on a FRESH random miss list every repetition (no list is
re-read), and reports the store's AnonHugePages from /proc/self/smaps.

    python scripts/gather_tlb.py            # M=126 misses per pool, 20 / 32 CTAs
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])  # a scratch variant build
from paper_2512_10576_b200.cache import AccessBatch, PoolSet  # noqa: E402
from paper_2512_10576_b200.transfer import HostLatentStore, gather  # noqa: E402

B, K = 64, 2048
M = int(os.environ.get("M", 126))
REPS = int(os.environ.get("REPS", 8))


def smaps_huge(addr: int, nbytes: int) -> int:
    """AnonHugePages (kB) of the mappings overlapping [addr, addr + nbytes)."""
    tot, inside = 0, False
    with open("/proc/self/smaps") as f:
        for line in f:
            head = line.split()[0]
            if "-" in head and ":" not in head:
                lo, hi = (int(x, 16) for x in head.split("-"))
                inside = lo < addr + nbytes and hi > addr
            elif inside and line.startswith("AnonHugePages:"):
                tot += int(line.split()[1])
    return tot


class PinnedStore:
    """Duck-typed store over a torch pinned (cudaHostAlloc) buffer: UVA, device ptr = host ptr."""

    def __init__(self, pools, rows):
        self.rows_per_pool, self.pitch = rows, _lib.HOST_ROW_PITCH
        self.buf = torch.empty(pools * rows * self.pitch, dtype=torch.uint8, pin_memory=True)
        self.device_ptr = self.buf.data_ptr()
        self.nbytes = self.buf.numel()

    def pool_ptr(self, begin):
        return self.device_ptr + begin * self.rows_per_pool * self.pitch


def run(hist: int, kind: str) -> None:
    cap = hist // 4
    pools = PoolSet(B, hist, cap, cap, row_bytes=1152)
    if kind == "pinned":
        store = PinnedStore(B, hist)
        huge = smaps_huge(store.device_ptr, store.nbytes)
    else:
        store = HostLatentStore(B, hist, hugepages=(kind == "thp"), vmm=(kind == "vmm"))
        assert store.vmm == (kind == "vmm"), "host VMM allocation fell back to the registered store"
        huge = smaps_huge(store._host_ptr, store.nbytes)
    g = torch.Generator(device="cuda").manual_seed(hist)
    z = lambda: torch.zeros((B, K), dtype=torch.int32, device="cuda")  # noqa: E731
    lists = []
    for _ in range(REPS + 2):
        acc = AccessBatch(counts=torch.zeros((B, 4), dtype=torch.int32, device="cuda"), sel_row=z(),
                          miss_ids=z(), miss_row=z(), hit_row=z())
        acc.counts[:, 1] = M
        acc.miss_ids[:, :M] = torch.rand((B, hist), device="cuda", generator=g).argsort(dim=1)[:, :M].int()
        acc.miss_row[:, :M] = torch.rand((B, cap), device="cuda", generator=g).argsort(dim=1)[:, :M].int()
        lists.append(acc)
    byt = B * M * 656
    for ctas in [int(c) for c in os.environ.get("CTAS", "20,32").split(",")]:
        gather(pools, store, lists[0], max_ctas=ctas)
        gather(pools, store, lists[1], max_ctas=ctas)
        torch.cuda.synchronize()
        ts = []
        for acc in lists[2:]:
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gather(pools, store, acc, max_ctas=ctas)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        med = ts[len(ts) // 2]
        print(f"hist={hist:6d} store={store.nbytes / 2**30:5.2f} GiB {kind:6s} AnonHuge={huge / 2**20:6.2f} GiB "
              f"ctas={ctas}: median {med:6.1f} us  {byt / med / 1e3:5.1f} GB/s useful  "
              f"(min {ts[0]:.1f}, max {ts[-1]:.1f})", flush=True)
    del store, pools, lists
    torch.cuda.synchronize()


for hist in [int(h) for h in os.environ.get("HISTS", "32768,131072").split(",")]:
    for kind in os.environ.get("KINDS", "thp,nothp,pinned,vmm").split(","):
        run(hist, kind)
