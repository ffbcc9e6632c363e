set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/quick_gpu.sh r2a rmat24 rmat22 rmat16 lattice2048 er4096
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a/bench_default.json 2> gpurun_out/r2a/bench_default.err; tail -c 3000 gpurun_out/r2a/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2a/launches.csv python bench.py --steps 2 --warmup 1 --cpu-baseline off > gpurun_out/r2a/ncu.log 2>&1; echo ncu=$?
