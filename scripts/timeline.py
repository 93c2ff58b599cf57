"""Device timeline of one DA-overlapped decode step (the schedule DSADecodeLayer.attend
captures), in us from the step start.  The whole step is queued behind a device sleep,
so host launch latency does not show: the numbers are the GPU's own critical path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_10576_b200.attention import SplitWorkspace, sparse_mla, sparse_mla_da  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer, ROW  # noqa: E402
from paper_2512_10576_b200.transfer import gather  # noqa: E402

B, ctx, rho = int(os.environ.get("B", 64)), int(os.environ.get("CTX", 32768)), float(os.environ.get("RHO", 0.25))
layer = DSADecodeLayer(B, ctx, rho, 2048, max_new_tokens=64, seed=5, drift=0.97)
layer.prefill_warmup(windows=8)
main = torch.cuda.current_stream()
side = torch.cuda.Stream(priority=-1)
adm = torch.cuda.Stream()
ws = SplitWorkspace(B, "cuda")
landed = torch.zeros(B, dtype=torch.int32, device="cuda")
rows = torch.zeros((B, 1, ROW), dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
layer.attend(*layer.next_queries())  # allocates the step buffers (layer.acc)
layer._append_device(rows)
layer.history += 1
for rep in range(int(os.environ.get("REPS", 12))):
    q_idx, q = layer.next_queries()
    torch.cuda.synchronize()
    torch.cuda._sleep(3_000_000)
    ev = {"start": E()}
    ev["start"].record(main)
    layer._select(q_idx, 0, B)
    acc = layer.acc
    ev["K1-K3"] = E(); ev["K1-K3"].record(main)
    adm.wait_event(ev["K1-K3"])
    with torch.cuda.stream(adm):
        layer._append_device(rows)
        ev["admit"] = E(); ev["admit"].record(adm)
    fused = bool(int(os.environ.get("FUSED", 1)))
    if not fused:
        landed.zero_()
    ev["zero"] = E(); ev["zero"].record(main)
    side.wait_event(ev["zero"])
    with torch.cuda.stream(side):
        gather(layer.pool, layer.store, acc, max_ctas=max(8, sms - 2 * B), exclusive=True,
               landed=landed if fused else None)
        ev["gather"] = E(); ev["gather"].record(side)
    if fused:
        sparse_mla_da(layer.pool, q, acc, landed, layer.sm_scale, out=layer.out, lse=layer.lse)
        ev["Attn"] = E(); ev["Attn"].record(main)
        main.wait_event(ev["gather"])
    else:
        sparse_mla(layer.pool, q, acc.hit_row, acc.counts[:, 0], layer.sm_scale, workspace=ws, mode="partial")
        ev["Attn0"] = E(); ev["Attn0"].record(main)
        main.wait_event(ev["gather"])
        sparse_mla(layer.pool, q, acc.miss_row, acc.counts[:, 1], layer.sm_scale, out=layer.out,
                   lse=layer.lse, workspace=ws, mode="resume")
        ev["Attn1"] = E(); ev["Attn1"].record(main)
    main.wait_event(ev["admit"])
    ev["end"] = E(); ev["end"].record(main)
    torch.cuda.synchronize()
    layer.history += 1
    if rep >= int(os.environ.get("REPS", 12)) - 3:
        print(" ".join(f"{k}={ev['start'].elapsed_time(e) * 1000:.1f}" for k, e in ev.items() if k != "start"),
              "misses", int(acc.counts[:, 1].sum()))
