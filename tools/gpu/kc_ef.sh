mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "coreness or synthetic or level_advance" > gpurun_out/kc_tests.log 2>&1; echo tests=$?
timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m > gpurun_out/kc_time.log 2>&1; echo time=$?
DG_B200_LIB=paper_2311_04333_b200/libdg_b200_noef.so timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m > gpurun_out/kc_time_noef.log 2>&1; echo time=$?
timeout 300 python tools/microbench.py > gpurun_out/microbench.log 2>&1; echo mb=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_coreness -c 1 python tools/kcore_time.py rmat26 > gpurun_out/kc26_dram.log 2>&1; echo ncu=$?
