mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:k_coreness -c 1 -o gpurun_out/kc22_new python tools/kcore_time.py rmat22 > gpurun_out/ncu_new.log 2>&1
DG_B200_LIB=paper_2311_04333_b200/$1 ncu --set full --clock-control none -k regex:k_coreness -c 1 -o gpurun_out/kc22_old python tools/kcore_time.py rmat22 > gpurun_out/ncu_old.log 2>&1
echo done
