#!/bin/bash
# Round-2 final records on the final code: GPU suite, C2 bench (with sub-records), C5,
# the reference arm, and the launch list of the bench command.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1; echo "suite exit=$?"
timeout 600 python bench.py > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo "bench exit=$?"
timeout 600 python bench.py --config c5 --no-sub --no-mtp > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "c5 exit=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err; echo "ref exit=$?"
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --target-processes application-only --log-file gpurun_out/final_launches_bench.csv python bench.py --quick --steps 3 --warmup 3 \
  > gpurun_out/final_launches_bench.log 2>&1; echo "launch list exit=$?"
