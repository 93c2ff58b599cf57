"""K1 alone at C2/C4 shapes: device time vs the persistent grid size (max_ctas), to see
how many SMs the HBM-bound indexer needs (the rest can host K2/K3/K4 concurrently).
Env: SHAPES="B:L,..." CTAS="148,..." FLUSH=1 (write 256 MB between runs: cold L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200 import _lib  # noqa: E402
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])  # a scratch variant build
from paper_2512_10576_b200.decode import _e4m3  # noqa: E402
from paper_2512_10576_b200.indexer import indexer_logits  # noqa: E402

SHAPES = [tuple(int(x) for x in t.split(":")) for t in
          os.environ.get("SHAPES", "64:32768,32:32768,64:131072").split(",")]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
for B, L in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    k = _e4m3(torch.randn((B, L, 128), device="cuda", generator=g) * 8)
    ks = torch.rand((B, L), device="cuda", generator=g) + 0.5
    q = _e4m3(torch.randn((B, 64, 128), device="cuda", generator=g) * 4)
    w = torch.randn((B, 64), device="cuda", generator=g) / 8
    lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
    out = torch.empty((B, L), device="cuda")
    byt = B * L * 136 + B * (64 * 128 + 256)
    for ctas in [int(c) for c in os.environ.get("CTAS", "148,128,112,96,80,64").split(",")]:
        for _ in range(3):
            indexer_logits(q, w, k, ks, lens, out=out, max_ctas=ctas)
        ts = []
        for _ in range(10):
            if flush is not None:
                flush.fill_(1)  # cold L2, as in the step
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); indexer_logits(q, w, k, ks, lens, out=out, max_ctas=ctas); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        print(f"{os.path.basename(_lib.LIB_PATH)} B={B} L={L} ctas={ctas}: {ts[5]:.1f} us  {byt / ts[5] / 1e3:.0f} GB/s")
    del k, ks, out
