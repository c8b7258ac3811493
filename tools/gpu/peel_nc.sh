mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "peel or run_golden or synthetic or medium" > gpurun_out/peel_tests.log 2>&1; echo tests=$?
timeout 600 python tools/peel_ab.py 26 10 0 > gpurun_out/peel26_flat.log 2>&1
timeout 600 python tools/peel_ab.py 22 20 0 > gpurun_out/peel22_flat.log 2>&1
