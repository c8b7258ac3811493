mkdir -p gpurun_out
for cfg in rmat22 rmat26; do
  timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_new.log 2>&1
  DG_KCORE_LOWLIST=0 timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_nolow.log 2>&1
  DG_B200_LIB=paper_2311_04333_b200/libdg_b200_kcold.so timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_old.log 2>&1
done
