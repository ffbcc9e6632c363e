O=gpurun_out/s5n; mkdir -p $O
for c in rmat24 rmat22; do python tools/variants.py run $c 3 ep1s32 ep1s64 ep1s128 ep1s256 ep1s64r1 2>&1 | tee $O/ab_$c.txt; done
