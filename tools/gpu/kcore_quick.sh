mkdir -p gpurun_out
timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m er_planted > gpurun_out/kc_time.log 2>&1; echo time=$?
timeout 300 python tools/kcore_probe.py rmat26 > gpurun_out/kcore_probe_rmat26.log 2>&1; echo probe=$?
timeout 300 python tools/kcore_probe.py rmat22 > gpurun_out/kcore_probe_rmat22.log 2>&1; echo probe=$?
timeout 300 python -m pytest tests -x -q -m gpu -k "coreness_golden or level_advance or without_alive" > gpurun_out/kc_tests.log 2>&1; echo tests=$?
