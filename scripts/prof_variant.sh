#!/bin/bash
# bash prof_variant.sh TAG LIB CONFIG MODE REGEX
TAG=$1; L=$2; CFG=$3; MODE=$4; RX=$5
mkdir -p gpurun_out
[ "$L" != default ] && export FVB_LIB_PATH=$L
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 3 -c 1 -o gpurun_out/${TAG}_full -f \
  python bench.py --config $CFG --mode $MODE --no-exact-leg --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_full.log 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
