"""Event timeline of one DA-overlapped decode step (eager, both streams), in us from
the step start — shows whether the side-stream gather overlaps attention pass 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_10576_b200.attention import SplitWorkspace, sparse_mla  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402
from paper_2512_10576_b200.indexer import indexer_logits, topk  # noqa: E402
from paper_2512_10576_b200.transfer import gather  # noqa: E402

B, ctx, rho = int(os.environ.get("B", 64)), int(os.environ.get("CTX", 32768)), float(os.environ.get("RHO", 0.25))
CTAS = int(os.environ.get("CTAS", 32))
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=32, seed=5, drift=0.97)
layer.prefill_warmup(windows=8)
main = torch.cuda.current_stream()
side = torch.cuda.Stream(priority=-1)
ws = SplitWorkspace(B, "cuda")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for rep in range(4):
    q_idx, q = layer.next_queries()
    torch.cuda.synchronize()
    ev = {"start": E()}
    ev["start"].record(main)
    indexer_logits(q_idx, layer.w, layer.k_cache, layer.k_scale, layer.lens, out=layer.logits)
    ev["K1"] = E(); ev["K1"].record(main)
    topk(layer.logits, layer.lens, 2048, out=layer.idx, count=layer.cnt)
    ev["K2"] = E(); ev["K2"].record(main)
    acc = layer.pool.access(layer.idx, layer.cnt)
    ev["K3"] = E(); ev["K3"].record(main)
    side.wait_event(ev["K3"])
    with torch.cuda.stream(side):
        ev["K4start"] = E(); ev["K4start"].record(side)
        gather(layer.pool, layer.store, acc, max_ctas=CTAS, exclusive=bool(int(os.environ.get("EXCL", 1))))
        ev["K4"] = E(); ev["K4"].record(side)
    sparse_mla(layer.pool, q, acc.hit_row, acc.counts[:, 0], layer.sm_scale, workspace=ws, mode="partial")
    ev["Attn0"] = E(); ev["Attn0"].record(main)
    main.wait_event(ev["K4"])
    ev["Attn1start"] = E(); ev["Attn1start"].record(main)
    sparse_mla(layer.pool, q, acc.miss_row, acc.counts[:, 1], layer.sm_scale, out=layer.out, lse=layer.lse,
               workspace=ws, mode="resume")
    ev["Attn1"] = E(); ev["Attn1"].record(main)
    layer.append_token()
    ev["append"] = E(); ev["append"].record(main)
    torch.cuda.synchronize()
    if rep == 3:
        for k, e in ev.items():
            print(f"{k:10s} {ev['start'].elapsed_time(e) * 1000:8.1f} us")
        print("misses", int(acc.counts[:, 1].sum()))
