O=gpurun_out/s5i; mkdir -p $O
for v in stats2 stats2s; do
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so python tools/profile_step.py rmat24 1 2>&1 | grep "CTA\|step" | tee -a $O/stats.txt
done
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_stats2.so python tools/profile_step.py rmat22 1 2>&1 | grep "CTA\|step" | tee -a $O/stats.txt
