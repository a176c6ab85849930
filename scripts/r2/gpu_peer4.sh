set -x
mkdir -p gpurun_out/peer4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:peer_boundary_kernel -c 1 -o gpurun_out/peer4/pbk python scripts/r2/peer_probe.py 4096 1 > gpurun_out/peer4/ncu.log 2>&1
tail -3 gpurun_out/peer4/ncu.log
timeout 600 python scripts/r2/nowait_probe.py 2>&1 | tail -5
timeout 600 python scripts/r2/nowait_probe.py nowait 2>&1 | tail -5
