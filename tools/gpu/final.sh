mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/gputest.log 2>&1; echo tests=$?
bash tools/gpu/profile_c4.sh
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c4.log 2>&1; echo ref=$?
timeout 1200 python tools/config_check.py rmat28 > gpurun_out/cc_rmat28.json 2> gpurun_out/cc_rmat28.err; echo cc28=$?
