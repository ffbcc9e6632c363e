O=gpurun_out/s5j; mkdir -p $O
python tools/variants.py run rmat24 3 cur c512 c2048 ur1 ur3 2>&1 | tee $O/knobs.txt
python tools/variants.py run rmat22 3 cur c512 c2048 2>&1 | tee -a $O/knobs.txt
