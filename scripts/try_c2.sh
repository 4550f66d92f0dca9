# On the GPU box: 2D parity tests + C2 timing of a variant library.   bash scripts/try_c2.sh lib.so|default
L=$1
if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "2d_warp or random_vs_oracle or full_size or at_rest" 2>&1 | tail -1
for c in c2 x2p17; do
timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$c', round(d['value']/1e9,2), 'kernel_us', round(r['kernel_ms']*1e3,1))"
done
