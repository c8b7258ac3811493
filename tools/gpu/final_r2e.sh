mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gputest.log 2>&1; echo tests=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_peel_cluster -c 2 -o gpurun_out/pc26 -f python tools/run_once.py rmat26 2 > gpurun_out/pc26_ncu.log 2>&1; echo ncu_pc=$?
for c in er_planted rmat22 chunglu50m; do timeout 900 python tools/config_check.py $c > gpurun_out/cc_$c.json 2> gpurun_out/cc_$c.err; echo $c=$?; done
