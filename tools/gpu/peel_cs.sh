mkdir -p gpurun_out
timeout 600 python tools/peel_ab.py 26 10 0 > gpurun_out/peel26_cs16.log 2>&1
DG_CLUSTER_CS=8 timeout 600 python tools/peel_ab.py 26 10 0 > gpurun_out/peel26_cs8.log 2>&1
DG_CLUSTER_CS=8 DG_CLUSTER_PT=1024 timeout 600 python tools/peel_ab.py 26 10 0 > gpurun_out/peel26_cs8_1024.log 2>&1
timeout 600 python tools/peel_ab.py 22 20 0 > gpurun_out/peel22_cs16.log 2>&1
DG_CLUSTER_CS=8 timeout 600 python tools/peel_ab.py 22 20 0 > gpurun_out/peel22_cs8.log 2>&1
