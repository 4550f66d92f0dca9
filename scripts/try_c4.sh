# On the GPU box: small3d parity tests + C4 timing of a variant library.   bash scripts/try_c4.sh lib.so|default
L=$1
if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "small3d or random_vs_oracle or at_rest or golden_drop_in" 2>&1 | tail -1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('c4', round(d['value']/1e9,2), 'kernel_us', round(r['kernel_ms']*1e3,1), d['clocks'])"
timeout 300 python bench.py --config x3p8 --steps 30 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('x3p8', round(d['value']/1e9,2), 'kernel_us', round(r['kernel_ms']*1e3,1))"
