mkdir -p gpurun_out
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_spprof.so timeout 600 python tools/sharded_persist_probe.py rmat22 1 4 > gpurun_out/sp_prof22.log 2>&1; echo probe=$?
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_spprof.so timeout 600 python tools/sharded_persist_probe.py rmat26 1 > gpurun_out/sp_prof26.log 2>&1; echo probe=$?
