#!/bin/bash
# On the GPU box: for each variant library given (or the default build), a quick
# bitwise parity check against the oracle and a device-timed bench line.
#   bash scripts/ab.sh CONFIG lib1.so lib2.so ...     (use "default" for the in-tree build)
CFG=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
  echo "=== $L ($CFG)"
  [ -n "$NOTEST" ] || timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "random_vs_oracle or golden_drop_in" 2>&1 | tail -1
  timeout 300 python bench.py --config $CFG --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || tail -5 /tmp/ab.err
  python - <<'PY'
import json
d = json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
r = d['roofline']
print(f"  value {d['value']/1e9:.2f} Gcell/s  kernel {r['kernel_ms']*1e3:.1f} us  frac {r['frac']:.3f}  clocks {d['clocks']}")
PY
done
