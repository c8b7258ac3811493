mkdir -p gpurun_out
set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c4.log 2>&1; echo ref=$?
DG_KCORE_PROFILE=1 timeout 300 python tools/kcore_probe.py rmat26 > gpurun_out/kcore_probe_rmat26.log 2>&1; echo probe=$?
