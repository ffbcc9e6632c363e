O=gpurun_out/s5m; mkdir -p $O
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_ep1s32.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_edge_prep -c 1 -o $O/prep python tools/profile_step.py rmat24 1 > $O/ncu.log 2>&1
ls -la $O
