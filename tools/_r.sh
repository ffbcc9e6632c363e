O=gpurun_out/s6c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_dist.py -m "gpu and not slow" -x -q 2>&1 | tail -2
for v in lr mi; do
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$v.csv python tools/profile_step.py rmat24 1 > $O/l_$v.log 2>&1
echo $v; python tools/ncu_summary.py launches $O/l_$v.csv 2>/dev/null | grep "k_build_up\|k_make_items"
done
for c in rmat24 rmat22 rmat16; do python tools/variants.py run $c 3 lr mi; done
