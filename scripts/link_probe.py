"""Host-link probe (python scripts/link_probe.py): H2D (10 MB queries), D2H (8.4 MB output), both at once, and the C2
miss gather alone / beside each copy."""
import os, sys, torch, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10576_b200.decode import DSADecodeLayer
from paper_2512_10576_b200.transfer import gather

dev = torch.device("cuda", 0)
hq = torch.empty(64 * 128 * 576 * 2, dtype=torch.uint8).pin_memory()
dq = torch.empty_like(hq, device=dev)
ho = torch.empty(64 * 128 * 512 * 2, dtype=torch.uint8).pin_memory()
do = torch.empty_like(ho, device=dev)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

layer = DSADecodeLayer(64, 32768, 0.25, 2048, max_new_tokens=64, seed=1234, drift=0.97)
layer.prefill_warmup(windows=32)
q_idx, q = layer.next_queries()
layer.attend(q_idx, q, overlap="none")
torch.cuda.synchronize()
acc = layer.acc
nmiss = int(acc.counts[:, 1].sum())
print("misses", nmiss, "MB", nmiss * 704 / 1e6)

def timed(fns, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        evs = []
        for st, fn in fns:
            st.wait_event(e0)
            with torch.cuda.stream(st):
                fn()
                ev = torch.cuda.Event(); ev.record(st); evs.append(ev)
        for ev in evs:
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]

h2d = lambda: dq.copy_(hq, non_blocking=True)
d2h = lambda: ho.copy_(do, non_blocking=True)
g = lambda: gather(layer.pool, layer.store, acc, max_ctas=20, exclusive=True)
g32 = lambda: gather(layer.pool, layer.store, acc, max_ctas=32, exclusive=True)
for name, fns in [("h2d", [(s1, h2d)]), ("d2h", [(s2, d2h)]), ("h2d+d2h", [(s1, h2d), (s2, d2h)]),
                  ("gather20", [(s3, g)]), ("gather32", [(s3, g32)]), ("gather20+d2h", [(s3, g), (s2, d2h)]),
                  ("gather20+h2d", [(s3, g), (s1, h2d)]), ("all3", [(s3, g), (s1, h2d), (s2, d2h)])]:
    us = timed(fns)
    print(f"{name:14s} {us:8.1f} us")
print("h2d GB/s", hq.numel() / timed([(s1, h2d)]) / 1e3, "d2h GB/s", ho.numel() / timed([(s2, d2h)]) / 1e3,
      "gather link GB/s", nmiss * 704 / timed([(s3, g)]) / 1e3)
