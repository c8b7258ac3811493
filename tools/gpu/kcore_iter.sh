mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "coreness or rmat22 or synthetic or level_advance or hepth or c1_" > gpurun_out/kc_tests.log 2>&1; echo tests=$?
timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m er_planted > gpurun_out/kc_time.log 2>&1; echo time=$?
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_nohub.so timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m > gpurun_out/kc_time_nohub.log 2>&1; echo time=$?
