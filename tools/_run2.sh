O=gpurun_out/s5b; mkdir -p $O
python tools/variants.py run rmat24 2 new noup nooff nostream noload 2>&1 | tee $O/attrib.txt
TCB_LIBRARY=paper_2403_02997_b200/lib/variants/libtricount_b200_stats.so python tools/profile_step.py rmat24 1 2>&1 | grep "CTA stats" | tee $O/stats.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_isect_cta -c 1 -o $O/cta_r24 python tools/profile_step.py rmat24 1 > $O/ncu_full.log 2>&1
ls -la $O
