mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench=$?
