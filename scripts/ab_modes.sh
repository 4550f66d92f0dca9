#!/bin/bash
# On the GPU box: exact / fast update times (scripts/time_modes.py) for each library
# given ("default" = the in-tree build), then the fast-mode and C3 parity tests on each.
#   bash scripts/ab_modes.sh CONFIG lib1.so lib2.so ...
CFG=$1; shift
for L in "$@"; do
  if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
  echo "=== $L ($CFG)"
  timeout 300 python scripts/time_modes.py --config $CFG --iters 30 2>&1 | tail -4
  [ -n "$NOTEST" ] || timeout 600 python -m pytest -q -x tests/test_gpu_fast.py tests/test_gpu_parity.py -k "fast or full_size or c3 or random_vs_oracle or golden" 2>&1 | tail -1
done
