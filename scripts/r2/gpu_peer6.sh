set -x
mkdir -p gpurun_out/peer6
timeout 900 python -m pytest tests/test_gpu_peer_strips.py tests/test_gpu_peer_ipc.py -q -x 2>&1 | tail -2
timeout 900 python scripts/r2/peer_scaling.py 2>&1 | tee gpurun_out/peer6/peer_scaling.log | tail -12
