#!/bin/bash
# Runs on the GPU box (via gpurun): ncu launch list of one bench command and
# one `--set full` capture of the fused kernel.  Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
CFG=${2:-c3}
LAYOUT=${3:-aos}
OUT=gpurun_out/prof_${TAG}_${CFG}_${LAYOUT}
mkdir -p gpurun_out
# launch list: every kernel of a short bench run with its device time
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file ${OUT}_launches.csv \
    python bench.py --config ${CFG} --layout ${LAYOUT} --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > ${OUT}_launches.log 2>&1
# one full capture of the fused update kernel (skip the first launches)
ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 \
    -o ${OUT}_full -f \
    python bench.py --config ${CFG} --layout ${LAYOUT} --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > ${OUT}_full.log 2>&1
echo done
