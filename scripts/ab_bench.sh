#!/bin/bash
# On the GPU box: bench.py device-timed lines (no e2e / CPU legs) for each library.
#   bash scripts/ab_bench.sh CONFIG MODE lib1.so lib2.so ...   ("default" = in-tree build)
CFG=$1; MODE=$2; shift 2
for L in "$@"; do
  if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
  timeout 300 python bench.py --config $CFG --mode $MODE --no-exact-leg --steps 200 --warmup 5 --e2e-steps 0 \
    --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || tail -5 /tmp/ab.err
  python - "$L" <<'PY'
import json, sys
d = json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
r = d['roofline']
print(f"{sys.argv[1].split('/')[-1]:28s} {d['value']/1e9:6.2f} Gcell/s  step {d['ms_per_step']*1e3:6.1f} us  kernel {r['kernel_ms']*1e3:6.1f} us  frac {r['frac']:.3f}  sm {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
PY
done
