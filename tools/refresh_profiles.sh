# Round-end measurement refresh (run on the GPU box): ncu launch list of the
# rmat24 step with per-kernel DRAM bytes (-> profiles/ncu_traffic.json), bench
# lines for every config, a full ncu capture of k_isect_cta, and DRAM bytes of
# every BFS/components kernel at rmat24 and the lattice.  Outputs under
# gpurun_out/$TAG; copy the summaries into profiles/.
set -x
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
python tools/profile_step.py rmat24 2 > $O/step_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_rmat24.csv python tools/profile_step.py rmat24 2 > $O/ncu_launch.log 2>&1
python tools/ncu_traffic.py $O/launches_rmat24.csv rmat24 profiles/ncu_traffic.json "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, python tools/profile_step.py rmat24 2 (last launch of each kernel), $TAG" > /dev/null
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python tools/ncu_summary.py launches $O/launches_rmat24.csv > $O/launches_rmat24.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_lattice.csv python tools/profile_step.py lattice2048 2 > $O/ncu_launch_lattice.log 2>&1
python tools/ncu_summary.py launches $O/launches_lattice.csv > $O/launches_lattice.txt
python bench.py > $O/bench_rmat24.json 2> $O/bench_rmat24.err; tail -c 600 $O/bench_rmat24.json
for c in rmat22 lattice2048 rmat16 er4096; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_isect_cta -c 1 -o $O/cta_r24 python tools/profile_step.py rmat24 1 > $O/ncu_full.log 2>&1
# the record pass, the warp tier, the UP build and the rank pass
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_edge_prep|k_isect_warp|k_build_up|k_rank_assign" -c 4 -o $O/prep_r24 python tools/profile_step.py rmat24 1 > $O/ncu_prep.log 2>&1
ls -la $O
# Back in the container (the .ncu-rep files come back in gpurun_out/$TAG):
#   python tools/ncu_profile_txt.py gpurun_out/$TAG/cta_r24.ncu-rep k_isect_cta \
#       paper_2403_02997_b200/lib/libtricount_b200.so > profiles/r02_ncu_isect_cta_rmat24.txt
#   python tools/ncu_profile_txt.py gpurun_out/$TAG/prep_r24.ncu-rep k_edge_prep   (etc.)
#   cp gpurun_out/$TAG/{ncu_traffic.json,bench_*.json,launches_*.txt} profiles/ (r02_ names)
