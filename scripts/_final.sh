bash scripts/gpu_check.sh > gpurun_out/final.log 2>&1
bash scripts/prof_r02.sh r02h_c3fast c3 fast fast3d_rpc r02h_c2fast c2 fast fused2d_warp > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1
