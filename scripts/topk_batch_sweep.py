"""K2 (ess_topk) latency vs batch at 32K rows (cold L2 between runs is not forced: the
logits of one micro-batch are L2-resident in the step too).  Env ESS_TOPK_MIN_CLUSTER
picks the cluster size (read once per process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200.indexer import topk  # noqa: E402

n, k = int(os.environ.get("CTX", 32768)), 2048
for B in (4, 8, 16, 48, 64):
    g = torch.Generator(device="cuda").manual_seed(0)
    logits = torch.randn((B, n), device="cuda", generator=g) * 3
    lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
    idx = torch.empty((B, k), dtype=torch.int32, device="cuda")
    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
    for _ in range(5):
        topk(logits, lens, k, out=idx, count=cnt)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); topk(logits, lens, k, out=idx, count=cnt); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"cluster>={os.environ.get('ESS_TOPK_MIN_CLUSTER', '1')} B={B:3d} n={n}: "
          f"median {ts[len(ts) // 2]:.1f} us  min {ts[0]:.1f} us", flush=True)
