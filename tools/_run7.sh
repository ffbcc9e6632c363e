O=gpurun_out/s5g; mkdir -p $O
python tools/variants.py run rmat24 2 small small1 big big1 2>&1 | tee $O/oneslice.txt
