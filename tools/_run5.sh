O=gpurun_out/s5e; mkdir -p $O
python tools/variants.py run rmat24 3 new mid mid86 mid4 midct256 2>&1 | tee $O/ab_rmat24.txt
