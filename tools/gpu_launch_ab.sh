# Per-kernel launch times of library variants: bash tools/gpu_launch_ab.sh TAG CONFIG NAME...
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out/$tag
for v in "$@"; do
  TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launch_${cfg}_$v.csv python tools/profile_step.py $cfg 2 > gpurun_out/$tag/launch_${cfg}_$v.log 2>&1
  echo "== $v"; python tools/ncu_summary.py launches gpurun_out/$tag/launch_${cfg}_$v.csv | head -16
done
