bash tools/refresh_profiles.sh r02g > gpurun_out/r02g_refresh.log 2>&1
O=gpurun_out/r02g
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_edge_prep|k_isect_warp|k_build_up|k_rank_assign" -c 4 -o $O/prep_r24 python tools/profile_step.py rmat24 1 > $O/ncu_prep.log 2>&1
bash tools/gpu_other_kernels.sh r02g > /dev/null 2>&1
ls $O | head -50
