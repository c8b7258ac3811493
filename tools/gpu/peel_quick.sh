mkdir -p gpurun_out
timeout 600 python tools/peel_ab.py 26 10 "$MODES" > gpurun_out/peel26.log 2>&1; echo ab26=$?
timeout 600 python tools/peel_ab.py 22 20 "$MODES" > gpurun_out/peel22.log 2>&1; echo ab22=$?
timeout 900 python -m pytest tests -x -q -m gpu -k "peel or run_golden or density or medium_rmat or c1_" > gpurun_out/peel_tests.log 2>&1; echo tests=$?
