mkdir -p gpurun_out/r2n
for v in seg2 flag2; do
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so timeout 600 ncu --set full --clock-control none -k regex:k_isect_cta -c 1 -o gpurun_out/r2n/cta22_$v python tools/profile_step.py rmat22 1 > gpurun_out/r2n/ncu_$v.log 2>&1
done
