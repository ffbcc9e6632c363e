# One GPU call during development: the GPU test suite, then short bench lines.
#   bash tools/quick_gpu.sh TAG [configs...]
tag=$1; shift
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$tag/pytest.log 2>&1; echo "pytest=$?"; tail -4 gpurun_out/$tag/pytest.log
for c in "${@:-rmat24}"; do
  timeout 300 python bench.py --config $c --cpu-baseline off > gpurun_out/$tag/bench_$c.json 2> gpurun_out/$tag/bench_$c.err
  python - "$c" "gpurun_out/$tag/bench_$c.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit(0)
st = d["stages_ms"]; r = d["roofline"]
print(f"{sys.argv[1]}: {d['ms_per_step']:.2f} ms/step  value={d['value']/1e9:.3f} Gedges/s  e2e={d['e2e']['value']/1e9:.3f}  "
      + " ".join(f"{k}={v:.2f}" for k, v in st.items() if v) + f"  cta_frac={r['frac']}")
PY
  tail -2 gpurun_out/$tag/bench_$c.err
done
