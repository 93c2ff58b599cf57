"""Small workloads of the kernels added in round 2's third session, for compute-sanitizer
(memcheck / racecheck / synccheck): the MTP path (indexer_kernel<2..4>, MTP top-k rows,
the MTP access with the per-set attention split, K5 over (request, token) rows in
partial / resume, per-request admission) under the none / DA / DBA schedules; the
streamed step (K1 request groups + done counters, the persistent top-k, the claim
gather; the sanitizer serialises kernels in launch order, which the hand-off protocol
tolerates); the f16 range guard (inf q: latched error, no hang)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_10576_b200.decode import DSADecodeLayer  # noqa: E402
from paper_2512_10576_b200.mtp import MTPDecodeLayer, draw_accepted  # noqa: E402

PARTS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["mtp", "stream", "range"]
rng = np.random.default_rng(0)
for mtp in ((1, 2, 3) if "mtp" in PARTS else ()):
    layer = MTPDecodeLayer(2, 16384, 0.5, 2048, mtp=mtp, max_new_tokens=6, seed=mtp, drift=0.9)
    layer.prefill_warmup(windows=2)
    for overlap in os.environ.get("OVERLAPS", "none,da,dba").split(","):
        acc = draw_accepted(rng, 2, 1.7, mtp + 1)
        q_idx, q = layer.next_queries(acc)
        layer.attend(q_idx, q, overlap=overlap)
        layer.append_tokens(acc)
    torch.cuda.synchronize()
    layer.pool.check("mtp")
    layer.close()
layer = DSADecodeLayer(2, [9000, 10500], 0.25, 2048, max_new_tokens=6, seed=2, drift=0.9)
layer.prefill_warmup(windows=2)
for _ in range(2 if "stream" in PARTS else 0):
    q_idx, q = layer.next_queries()
    layer.attend(q_idx, q, overlap="stream")
    layer.append_token()
torch.cuda.synchronize()
layer.pool.check("stream")
if "range" in PARTS:
    q_idx, q = layer.next_queries()
    q[1, 5, 3] = float("inf")
    layer.attend(q_idx, q, overlap="none")
    torch.cuda.synchronize()
    try:
        layer.pool.check("range")
        raise SystemExit("range guard did not fire")
    except ValueError as e:
        print("range guard:", e)
layer.close()
print("sanitize_r02 ok")
