# A/B of library variants in one GPU session: bash tools/gpu_ab.sh TAG CONFIG STEPS NAME...
tag=$1; cfg=$2; steps=$3; shift 3
mkdir -p gpurun_out/$tag
for i in 1 2; do python tools/variants.py run $cfg $steps "$@"; done 2>&1 | tee gpurun_out/$tag/ab_$cfg.txt
