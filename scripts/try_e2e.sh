# On the GPU box: host-pipeline parity tests + e2e of C3/C2/C4 for a variant library.  bash scripts/try_e2e.sh lib|default
L=$1
if [ "$L" = default ]; then unset FVB_LIB_PATH; else export FVB_LIB_PATH=$L; fi
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "odd_chunks or golden_drop_in or variant_equivalence" 2>&1 | tail -1
for c in c3 c2 c4; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('$c e2e', round(e['value']/1e9,3), round(e['roofline']['frac'],3))"
done
