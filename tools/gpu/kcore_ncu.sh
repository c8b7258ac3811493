mkdir -p gpurun_out
timeout 300 python tools/kcore_time.py rmat22 rmat26 chunglu50m er_planted > gpurun_out/kc_time.log 2>&1; echo time=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_coreness -c 1 -o gpurun_out/kc26 -f python tools/kcore_time.py rmat26 > gpurun_out/kc26_ncu.log 2>&1; echo ncu=$?
