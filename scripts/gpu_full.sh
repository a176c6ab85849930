set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dwt53 -s 2 -c 1 -o gpurun_out/prof_c3_v1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
