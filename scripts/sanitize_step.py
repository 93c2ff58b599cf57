"""Small decode workload for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
B = int(os.environ.get("B", 2))
layer = DSADecodeLayer(B, 4096, 0.25, 2048, max_new_tokens=8, seed=1, drift=0.9)
layer.prefill_warmup(windows=2)
for overlap in ("none", "da"):
    q_idx, q = layer.next_queries()
    layer.attend(q_idx, q, overlap=overlap)
    layer.append_token()
torch.cuda.synchronize()
layer.pool.check()
print("sanitize workload done")
