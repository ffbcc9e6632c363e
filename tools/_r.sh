O=gpurun_out/s5z; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_dist.py -m "gpu and not slow" -x -q 2>&1 | tail -3
for c in rmat24 rmat22 rmat16; do python tools/variants.py run $c 3 prev wrec; done
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_wrec.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l.csv python tools/profile_step.py rmat24 1 > $O/l.log 2>&1
python tools/ncu_summary.py launches $O/l.csv 2>/dev/null | grep "k_edge_prep\|k_isect_warp\|k_isect_cta"
