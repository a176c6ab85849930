mkdir -p gpurun_out
timeout 900 python scripts/scheme_compare.py --iters 30 > gpurun_out/scheme_compare.log 2>&1; tail -8 gpurun_out/scheme_compare.log
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1; tail -12 gpurun_out/inverse_bench.log
