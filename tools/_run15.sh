O=gpurun_out/s5o; mkdir -p $O
for g in 32 64 128; do echo "granularity $g"; TCB_L2_FETCH=$g python tools/variants.py run rmat24 3 l2g l2g0 2>&1; done | tee $O/l2.txt
python tools/variants.py run rmat24 3 l2g l2g0 2>&1 | tee -a $O/l2.txt
