set -x
mkdir -p gpurun_out/peer3
timeout 900 python -m pytest tests/test_gpu_peer_strips.py -q -x 2>&1 | tail -4
timeout 300 python scripts/r2/peer_probe.py 4096 1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/peer3/launches_sys.csv python scripts/r2/peer_probe.py 4096 1 > gpurun_out/peer3/ncu.log 2>&1
timeout 300 python scripts/r2/peer_probe.py 4096 1 peergpu && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/peer3/launches_gpu.csv python scripts/r2/peer_probe.py 4096 1 peergpu > gpurun_out/peer3/ncu2.log 2>&1
tail -3 gpurun_out/peer3/ncu.log gpurun_out/peer3/ncu2.log
