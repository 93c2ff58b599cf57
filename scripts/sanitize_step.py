"""Small decode workloads for compute-sanitizer (memcheck / racecheck / synccheck):
the oversize path (ctx 4K, cap 1024 < K) and the normal path (mixed 9K-13K contexts,
early admission), each under the none / DA / DBA schedules; small batches take the
split fused K5 + combine; plus the bulk-copy gather variant.  45K-131K rows run the
2- and 4-CTA cluster top-k (DSMEM histogram pushes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_10576_b200 import transfer  # noqa: E402
from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402

B = int(os.environ.get("B", 2))
for ctx in (4096, [9000 + 1500 * b for b in range(B)], [45000 + 5000 * b for b in range(B)],
            [100000 + 31072 * b for b in range(B)]):
    layer = DSADecodeLayer(B, ctx, 0.25, 2048, max_new_tokens=8, seed=1, drift=0.9)
    layer.prefill_warmup(windows=2)
    for overlap in ("none", "da", "dba"):
        q_idx, q = layer.next_queries()
        layer.attend(q_idx, q, overlap=overlap)
        layer.append_token()
    transfer.GATHER_BULK = True
    q_idx, q = layer.next_queries()
    layer.attend(q_idx, q, overlap="none")
    layer.append_token()
    transfer.GATHER_BULK = False
    torch.cuda.synchronize()
    layer.pool.check()
    layer.close()
print("sanitize workload done")
