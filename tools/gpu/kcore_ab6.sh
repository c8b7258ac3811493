mkdir -p gpurun_out
for cfg in rmat22 rmat26 chunglu50m; do
  timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_new.log 2>&1
  for v in noslot smallsm kcold; do
  DG_B200_LIB=paper_2311_04333_b200/libdg_b200_$v.so timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_$v.log 2>&1
  done
done
