#!/bin/bash
# On the GPU box: one `ncu --set full` capture of the fused update kernel of CONFIG
# (source-level stall attribution needs -lineinfo, which the Makefile sets).
#   bash scripts/ncu_full.sh TAG CONFIG [KERNEL_REGEX]
TAG=$1; CFG=${2:-c3}; RX=${3:-fused}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$RX -s 2 -c 1 -o gpurun_out/${TAG}_full -f \
  python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --config $CFG --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_launches.log 2>&1
ls -la gpurun_out
