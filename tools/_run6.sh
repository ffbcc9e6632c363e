O=gpurun_out/s5f; mkdir -p $O
for v in mid midns; do
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$v.csv python tools/profile_step.py rmat24 1 > $O/l_$v.log 2>&1
python tools/ncu_summary.py launches $O/l_$v.csv | grep -i "isect" 
done
