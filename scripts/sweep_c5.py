"""C5 sweep (BASELINE configs[4]): mixed 8K-128K batch, GPU slot-pool ratio x query drift
(the drift sets the step-to-step selection overlap and so the hit rate).  Each point is
one `bench.py --config c5 --quick` process; writes gpurun_out/c5_sweep.json."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rhos = [float(x) for x in os.environ.get("RHOS", "0.1,0.25,0.5").split(",")]
drifts = [float(x) for x in os.environ.get("DRIFTS", "0.9,0.97,0.99").split(",")]
rows = []
for rho in rhos:
    for dr in drifts:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5", "--quick",
                            "--rho", str(rho), "--drift", str(dr), "--steps", "10", "--warmup", "3"],
                           capture_output=True, text=True, timeout=900)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print("failed", rho, dr, r.stderr[-500:])
            continue
        rows.append({"sparse_ratio": rho, "drift": dr, "us_per_step": d["ms_per_step"] * 1e3,
                     "tokens_per_s": d["value"], "hit_rate": d["hit_rate"]})
        print(f"rho={rho:.2f} drift={dr:.2f}: {d['ms_per_step'] * 1e3:7.1f} us/step "
              f"{d['value']:9.0f} tok/s hit {d['hit_rate']:.4f}", flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "c5_sweep.json"), "w") as f:
    json.dump(rows, f, indent=1)
