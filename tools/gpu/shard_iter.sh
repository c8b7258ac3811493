mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py -x -q -m gpu -k "persistent" > gpurun_out/sp_tests.log 2>&1; echo tests=$?
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_spprof.so timeout 600 python tools/sharded_persist_probe.py rmat22 1 4 > gpurun_out/sp_prof22.log 2>&1; echo probe=$?
timeout 600 python tools/sharded_persist_probe.py rmat22 1 2 4 8 > gpurun_out/sp_probe22.log 2>&1; echo probe=$?
timeout 600 python tools/sharded_persist_probe.py rmat26 1 4 8 > gpurun_out/sp_probe26.log 2>&1; echo probe=$?
