bash scripts/gpu_check.sh
bash scripts/prof_r02.sh r02e_c4fast c4 fast small3d_kernel r02e_c3exact c3 exact fused3d_half
