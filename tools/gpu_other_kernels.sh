# ncu summaries of the kernels off the CTA tier: the small-graph kernel
# (ER-4096), the low-degree count (lattice), the warp tier and UP build (RMAT-24)
O=gpurun_out/${1:-r02o}; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:k_small_cetc -c 1 -o $O/small_er python tools/profile_step.py er4096 1 > $O/ncu_small.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_lowdeg_count -c 1 -o $O/lowdeg_lat python tools/profile_step.py lattice2048 1 > $O/ncu_lowdeg.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_isect_warp|k_build_up|k_owner_bits" -c 3 -o $O/prep_r24 python tools/profile_step.py rmat24 1 > $O/ncu_prep.log 2>&1
ls $O
