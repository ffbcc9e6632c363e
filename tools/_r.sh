O=gpurun_out/s5y; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_dist.py -m "gpu and not slow" -x -q 2>&1 | tail -3
for v in flat flat5; do
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$v.csv python tools/profile_step.py rmat24 1 > $O/l_$v.log 2>&1
echo $v; python tools/ncu_summary.py launches $O/l_$v.csv 2>/dev/null | grep "k_edge_prep\|k_scatter_off\|k_isect_cta"
done
for c in rmat24 rmat22 rmat16; do python tools/variants.py run $c 3 epm5 flat; done
