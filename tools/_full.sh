O=gpurun_out/s5t; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest=$?"; tail -4 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --cpu-baseline off > $O/bench_rmat24.json 2> $O/bench_rmat24.err; tail -c 1500 $O/bench_rmat24.json; tail -3 $O/bench_rmat24.err
