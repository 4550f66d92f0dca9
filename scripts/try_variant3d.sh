# On the GPU box: parity (random / full-size / edge-case tests vs the oracle) + C3 timing of a variant library.
#   bash scripts/try_variant3d.sh path/to/lib.so|default
L=$1
if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "random_vs_oracle or full_size or at_rest or signed_zero" 2>&1 | tail -2
timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('c3', round(d['value']/1e9,2), 'kernel_us', round(r['kernel_ms']*1e3,1), d['clocks'])"
