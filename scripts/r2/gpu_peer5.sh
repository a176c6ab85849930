set -x
mkdir -p gpurun_out/peer5
timeout 900 python -m pytest tests/test_gpu_peer_strips.py -q -x 2>&1 | tail -3
timeout 300 python scripts/r2/peer_probe.py 4096 1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/peer5/launches_probe.csv python scripts/r2/peer_probe.py 4096 1 > gpurun_out/peer5/ncu.log 2>&1
timeout 900 python scripts/r2/peer_scaling.py 2>&1 | tee gpurun_out/peer5/peer_scaling.log | tail -12
for c in 2 4; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/peer5/fwd53_c$c.json 2>&1; tail -c 250 gpurun_out/peer5/fwd53_c$c.json; echo; done
