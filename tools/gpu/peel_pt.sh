mkdir -p gpurun_out
DG_CLUSTER_PT=512 timeout 600 python tools/peel_ab.py 26 2 0 > gpurun_out/peel26_pt512.log 2>&1
