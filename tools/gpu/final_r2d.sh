mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2> gpurun_out/bench_c4.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_peel_cluster -c 2 -o gpurun_out/pc26 -f python tools/run_once.py rmat26 2 > gpurun_out/pc26_ncu.log 2>&1; echo ncu_pc=$?
timeout 1200 python tools/config_check.py rmat28 > gpurun_out/cc_rmat28.json 2> gpurun_out/cc_rmat28.err; echo cc28=$?
timeout 1200 python tools/config_check.py rmat26 > gpurun_out/cc_rmat26.json 2> gpurun_out/cc_rmat26.err; echo cc26=$?
