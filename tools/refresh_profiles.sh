# Round-end measurement refresh (run on the GPU box): bench lines, reference arm, ncu launch list, full ncu capture of k_isect_cta.
set -x
mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench_rmat24.json 2> gpurun_out/r01/bench_rmat24.err; tail -c 1500 gpurun_out/r01/bench_rmat24.json
for c in rmat22 lattice2048 rmat16 er4096; do python bench.py --config $c > gpurun_out/r01/bench_$c.json 2> gpurun_out/r01/bench_$c.err; done
python bench.py --impl reference > gpurun_out/r01/bench_reference.json 2> gpurun_out/r01/bench_reference.err
python tools/profile_step.py rmat24 2 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01/launches_rmat24.csv python tools/profile_step.py rmat24 2 > gpurun_out/r01/ncu_launch.log 2>&1
python tools/profile_step.py rmat24 1 && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_isect_cta -c 1 -o gpurun_out/r01/cta_r24 python tools/profile_step.py rmat24 1 > gpurun_out/r01/ncu_full.log 2>&1
ls -la gpurun_out/r01
