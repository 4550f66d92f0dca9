# ncu --set full of the 2D run_simulation fast-path kernels (scripts/time_direct2d.py: C2's 256^2 grid)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"halo_shell2d|totals_haloed_rows" -c 2 \
  -o gpurun_out/direct2d -f python scripts/time_direct2d.py > gpurun_out/ncu_direct2d.log 2>&1
tail -2 gpurun_out/ncu_direct2d.log
