# A/B of the k-core: current library vs a tuning build (DG_B200_LIB=$1)
mkdir -p gpurun_out
for cfg in rmat22 rmat26 chunglu50m; do
  timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_new.log 2>&1
  DG_B200_LIB=paper_2311_04333_b200/$1 timeout 300 python tools/kcore_time.py $cfg >> gpurun_out/ab_old.log 2>&1
done
timeout 300 python tools/kcore_probe.py rmat22 > gpurun_out/probe22_new.log 2>&1
DG_B200_LIB=paper_2311_04333_b200/$1 timeout 300 python tools/kcore_probe.py rmat22 > gpurun_out/probe22_old.log 2>&1
echo done
