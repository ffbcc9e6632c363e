mkdir -p gpurun_out/cap
timeout 900 python tools/scale_probe.py rmat25 2>&1 | tail -2 | tee gpurun_out/cap/cap.txt
timeout 900 python tools/scale_probe.py rmat26 2>&1 | tail -3 | tee -a gpurun_out/cap/cap.txt
