mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "coreness or rmat22 or synthetic or level_advance or hepth or c1_ or c4_ or c3_" > gpurun_out/kc_tests.log 2>&1; echo tests=$?
timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m er_planted > gpurun_out/kc_time.log 2>&1; echo time=$?
timeout 300 python tools/kcore_probe.py rmat26 > gpurun_out/kcore_probe_rmat26.log 2>&1; echo probe=$?
