O=gpurun_out/s5d; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -m "gpu and not slow" -x -q 2>&1 | tail -5
for i in 1 2; do python tools/variants.py run rmat24 3 new mid; done 2>&1 | tee $O/ab_rmat24.txt
python tools/variants.py run rmat22 3 base new mid 2>&1 | tee $O/ab_rmat22.txt
python tools/variants.py run rmat16 3 base new mid 2>&1 | tee $O/ab_rmat16.txt
