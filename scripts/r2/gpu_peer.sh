# Peer-memory halo strips: GPU tests, the emulated per-rank cost, the N=1 bench still intact
set -x
mkdir -p gpurun_out/peer
timeout 900 python -m pytest tests/test_gpu_peer_strips.py -q -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_strip_levels.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python scripts/r2/peer_scaling.py 2>&1 | tee gpurun_out/peer/peer_scaling.log | tail -20
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/peer/default_c3.json 2>&1; tail -c 400 gpurun_out/peer/default_c3.json
