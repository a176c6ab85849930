mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_inverse.py -q -x 2>&1 | tail -4
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1; cut -c1-420 gpurun_out/inverse_bench.log
