set -x
mkdir -p gpurun_out/peer2
timeout 900 python -m pytest tests/test_gpu_peer_strips.py -q -x 2>&1 | tail -4
timeout 900 python scripts/r2/peer_scaling.py 2>&1 | tee gpurun_out/peer2/peer_scaling.log | tail -20
timeout 300 python scripts/r2/peer_probe.py 4096 1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/peer2/launches_probe.csv python scripts/r2/peer_probe.py 4096 1 > gpurun_out/peer2/ncu.log 2>&1
tail -3 gpurun_out/peer2/ncu.log
