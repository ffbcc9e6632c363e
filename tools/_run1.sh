mkdir -p gpurun_out/s5a
python tools/profile_step.py rmat16 1 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -5
for i in 1 2; do python tools/variants.py run rmat24 3 base new; done 2>&1 | tee gpurun_out/s5a/ab_rmat24.txt
timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -x -q 2>&1 | tail -5
