# Re-entry check of the restored checkpoint: smoke, the GPU suite, the default bench line
set -x
mkdir -p gpurun_out/reentry
timeout 300 python __graft_entry__.py smoke
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/reentry/default_c3.json 2> gpurun_out/reentry/default_c3.err; tail -c 600 gpurun_out/reentry/default_c3.json
timeout 600 python bench.py --config 4 > gpurun_out/reentry/fwd53_c4.json 2> gpurun_out/reentry/fwd53_c4.err; tail -c 300 gpurun_out/reentry/fwd53_c4.json
