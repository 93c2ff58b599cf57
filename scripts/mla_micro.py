"""Time K5 (sparse MLA) alone at the C2 shape: B=64, 2048 of 8192 slot rows each.
FMT=656 (raw FP8 slot rows, the CTA-pair kernel) or 1152 (f16 slot rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_10576_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])  # a scratch variant build
from paper_2512_10576_b200.attention import SplitWorkspace, sparse_mla
from paper_2512_10576_b200.cache import PoolSet

B, cap, n = 64, 8192, int(os.environ.get("N", 2048))
MODE = os.environ.get("MODE", "full")
FMT = int(os.environ.get("FMT", "656"))
pools = PoolSet(B, 32768, cap, cap, row_bytes=FMT)
g = torch.Generator(device="cuda").manual_seed(0)
rv = pools.rows_view()
if FMT == 656:
    from paper_2512_10576_b200.decode import random_latent_rows
    for b in range(B):
        rv[b].copy_(random_latent_rows(cap, "cuda", g))
else:
    rv.copy_((torch.randn(rv.shape, device="cuda", generator=g) * 0.5).half())
sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:n] for _ in range(B)]).int()
cnt = torch.full((B,), n, dtype=torch.int32, device="cuda")
q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
out, lse = sparse_mla(pools, q, sel, cnt)
ws = SplitWorkspace(B, "cuda")
sparse_mla(pools, q, sel, cnt, workspace=ws, mode="partial")
run = lambda: sparse_mla(pools, q, sel, cnt, out=out, lse=lse, workspace=ws if MODE != "full" else None,
                         mode=MODE)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(int(os.environ.get("ITERS", "10"))):
    flush.zero_()
    torch.cuda._sleep(1_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
byt = B * n * FMT
print(f"{os.path.basename(_lib.LIB_PATH)} sparse_mla fmt={FMT} {MODE} B={B} n={n}: median {ts[len(ts)//2]:.1f} us, min {ts[0]:.1f} us, "
      f"{byt / ts[len(ts)//2] / 1e3:.0f} GB/s unique rows")
