# pyramid launches: parity + config 4 / 4b / 5 timing + launch list
set -x
mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_odd_pitch.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -5
for c in 4 4b 5 2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2b/fwd53_c$c.json 2> gpurun_out/r2b/fwd53_c$c.err; tail -c 400 gpurun_out/r2b/fwd53_c$c.json; tail -3 gpurun_out/r2b/fwd53_c$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2b/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 > /dev/null 2>&1; grep -c pyramid gpurun_out/r2b/launches_c4.csv
