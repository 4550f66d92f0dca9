# ncu --set full of the first halo_project launches of scripts/time_halo.py (3D p=16 on C3's grid)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:halo -c 2 -o gpurun_out/halo -f python scripts/time_halo.py > gpurun_out/ncu_halo.log 2>&1
tail -3 gpurun_out/ncu_halo.log
