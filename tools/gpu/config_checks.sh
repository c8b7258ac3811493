mkdir -p gpurun_out
for c in er_planted rmat22 chunglu50m rmat26 rmat28; do
  timeout 1200 python tools/config_check.py $c > gpurun_out/cc_$c.json 2> gpurun_out/cc_$c.err; echo $c=$?
done
