#!/bin/bash
# Round 2: FP8-slot K5 (CTA pair) vs the f16-slot K5, alone and in the product step;
# ncu captures of the FP8 K5 and of K4 with host-link (PCIe) counters.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for f in 656 1152; do FMT=$f timeout 120 python scripts/mla_micro.py; done
for f in fp8 f16; do
  ESS_SLOT_FORMAT=$f timeout 300 python bench.py --quick --steps 20 --warmup 5 | tail -1
  ESS_SLOT_FORMAT=$f timeout 300 python bench.py --quick --steps 20 --warmup 5 --config c4 | tail -1
done
FMT=656 timeout 600 $NCU --set full --clock-control none --import-source on -k regex:sparse_mla_fp8 -s 3 -c 1 \
  -o gpurun_out/prof_k5fp8 -f python scripts/mla_micro.py > gpurun_out/prof_k5fp8.log 2>&1; echo "ncu k5 rc=$?"
FMT=656 CTAS=20 M=120 timeout 600 $NCU --clock-control none -k regex:gather_kernel -s 3 -c 1 \
  --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_aperture_sysmem_op_read.sum,lts__t_sectors_aperture_sysmem_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/ncu_gather_pcie.csv python scripts/gather_micro.py > gpurun_out/ncu_gather.log 2>&1; echo "ncu gather rc=$?"
