bash tools/gpu_ab.sh r2c rmat24 3 base cut
bash tools/gpu_ab.sh r2c rmat22 3 base cut
bash tools/quick_gpu.sh r2c rmat24 rmat22 rmat16 lattice2048 er4096
