mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_build.py tests/test_sharded.py -x -q -m gpu > gpurun_out/dist_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --sharded --config rmat22 --steps 2 --warmup 1 > gpurun_out/bench_sharded22.log 2>&1; echo bench=$?
timeout 900 python bench.py --sharded --config rmat26 --steps 2 --warmup 1 > gpurun_out/bench_sharded26.log 2>&1; echo bench=$?
