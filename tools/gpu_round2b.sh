# sweep tests, fresh ncu full capture of k_isect_cta, the reference arm at rmat24
set -x
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > $O/sweep.log 2>&1; echo sweep=$?; tail -5 $O/sweep.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_isect_cta -c 1 -o $O/cta_r24 python tools/profile_step.py rmat24 1 > $O/ncu_full.log 2>&1; echo ncu=$?
( time timeout 1500 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err ) 2> $O/ref_time.txt; echo ref=$?; cat $O/ref_time.txt; tail -c 1500 $O/bench_reference.json
