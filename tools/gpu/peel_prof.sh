mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "peel or run_golden or synthetic or medium" > gpurun_out/peel_tests.log 2>&1; echo tests=$?
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_pprof.so timeout 600 python tools/cluster_probe2.py 26 1 3 > gpurun_out/cp26.log 2>&1; echo cp=$?
timeout 600 python tools/peel_ab.py 26 10 0,1 > gpurun_out/peel26_modes.log 2>&1; echo ab=$?
DG_NO_SLICE_SMEM=1 timeout 600 python tools/peel_ab.py 26 10 0 > gpurun_out/peel26_noslice.log 2>&1; echo ab=$?
