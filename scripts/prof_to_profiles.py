"""gpurun_out/prof_*.ncu-rep -> profiles/<ROUND>_ncu_<kernel>.txt (SOL excerpt + key raw
metrics; ROUND env, default r01) and profiles/traffic_<config>.json (K1 DRAM bytes per
launch, read by bench.py)."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
SOL = ("Memory Throughput", "DRAM Throughput", "Duration", "L2 Cache Throughput", "Compute (SM) Throughput",
       "Registers Per Thread", "Grid Size", "Block Size", "Achieved Occupancy", "Dynamic Shared Memory Per Block")
ALGO = {  # algorithmic bytes per launch at the prof_step shapes (B=64, len = ctx + steps)
    "indexer_kernel": lambda L: 64 * L * 136 + 64 * (64 * 128 + 256),
}
RND = os.environ.get("ROUND", "r01")
for name in sys.argv[1:]:
    rep = os.path.join(OUT, f"prof_{name}.ncu-rep")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    lines = [ln for ln in det.splitlines() if ln.strip().startswith(SOL) or "Section: GPU Speed Of Light" in ln]
    raw = summary(rep)[0]
    with open(os.path.join(PROF, f"{RND}_ncu_{name}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, {name} (scripts/gpu_prof_round.sh; one steady-state launch)\n")
        f.write("\n".join(lines[:14]) + "\n# raw metrics\n")
        for k, (v, u) in ((k, v) for k, v in raw.items() if k != "name"):
            f.write(f"  {k}: {v} {u}\n")
    if name.startswith("indexer_kernel"):
        cfg = "c4" if name.endswith("c4") else "c2"
        L = (131072 if cfg == "c4" else 32768) + 3
        rd, wr = float(raw["dram__bytes_read.sum"][0]), float(raw["dram__bytes_write.sum"][0])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(raw["dram__bytes_read.sum"][1], 1)
        wr *= scale.get(raw["dram__bytes_write.sum"][1], 1)
        dur = float(raw["gpu__time_duration.sum"][0]) * (1e-3 if raw["gpu__time_duration.sum"][1] == "ns" else 1)
        with open(os.path.join(PROF, f"traffic_{cfg}.json"), "w") as f:
            json.dump({"kernel": "indexer_kernel", "config": f"{cfg.upper()}: B=64 (+step headroom)",
                       "source": f"ncu --set full, gpurun_out/prof_{name}.ncu-rep ({RND})",
                       "indexer_dram_bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd),
                       "dram_write_bytes": int(wr), "algorithmic_bytes_per_launch": ALGO["indexer_kernel"](L),
                       "duration_us_ncu": dur}, f, indent=1)
    print(name, "ok")
