O=gpurun_out/s5l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -m "gpu and not slow" -x -q 2>&1 | tail -3
for c in rmat24 rmat22; do python tools/variants.py run $c 3 cur ep1 ep0 ep1s8 ep1s32 ep1s0 ep0s32 2>&1 | tee $O/ab_$c.txt; done
