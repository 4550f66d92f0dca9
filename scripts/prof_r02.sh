#!/bin/bash
# On the GPU box: launch list + one `ncu --set full` capture of the update kernel per
# (tag, config, mode, kernel-regex) tuple.  Outputs in gpurun_out/.
#   bash scripts/prof_r02.sh TAG CONFIG MODE REGEX [TAG CONFIG MODE REGEX ...]
mkdir -p gpurun_out
while [ $# -ge 4 ]; do
  TAG=$1; CFG=$2; MODE=$3; RX=$4; shift 4
  OUT=gpurun_out/${TAG}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${OUT}_launches.csv \
    python bench.py --config $CFG --mode $MODE --no-exact-leg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > ${OUT}_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 3 -c 1 -o ${OUT}_full -f \
    python bench.py --config $CFG --mode $MODE --no-exact-leg --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > ${OUT}_full.log 2>&1
  ncu -i ${OUT}_full.ncu-rep --page source --csv > ${OUT}_source.csv 2>/dev/null
done
ls -la gpurun_out
