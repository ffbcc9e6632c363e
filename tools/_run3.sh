O=gpurun_out/s5c; mkdir -p $O
python tools/variants.py run rmat24 2 new small big wt512 wt128 2>&1 | tee $O/attrib.txt
