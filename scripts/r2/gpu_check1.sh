# Round 2, first check: new tests + the bench with gate / step stats on configs 3, 2, 4, 5
set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_strip_levels.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -5
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
for c in 3 2 4 5 1; do
  timeout 600 python bench.py --config $c > gpurun_out/r2a/fwd53_c$c.json 2> gpurun_out/r2a/fwd53_c$c.err; tail -c 3000 gpurun_out/r2a/fwd53_c$c.json
done
timeout 600 python bench.py --impl reference > gpurun_out/r2a/ref_c3.json 2>&1; tail -c 1500 gpurun_out/r2a/ref_c3.json
timeout 600 python bench.py --config 3 --op inverse > gpurun_out/r2a/inv53_c3.json 2>&1; tail -c 600 gpurun_out/r2a/inv53_c3.json
timeout 600 python bench.py --config 3 --wavelet cdf97 --op inverse > gpurun_out/r2a/inv97_c3.json 2>&1; tail -c 600 gpurun_out/r2a/inv97_c3.json
timeout 600 python bench.py --config 4 --wavelet cdf97 > gpurun_out/r2a/fwd97_c4.json 2>&1; tail -c 600 gpurun_out/r2a/fwd97_c4.json
