# Round-end style check on one B200: GPU tests, smoke, the default bench line,
# the reference arm, every config, the scheme comparison, the inverse bench and
# the parity report (outputs under gpurun_out/).
set -x
mkdir -p gpurun_out
timeout 2800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; [ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 120 python __graft_entry__.py smoke
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
for c in 1 2 4 4b 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -1 gpurun_out/bench_c$c.json
done
for c in 3 4; do
  timeout 600 python bench.py --config $c --wavelet cdf97 > gpurun_out/bench97_c$c.json 2> gpurun_out/bench97_c$c.err; tail -1 gpurun_out/bench97_c$c.json
done
timeout 900 python scripts/scheme_compare.py > gpurun_out/scheme_compare.log 2>&1; tail -8 gpurun_out/scheme_compare.log
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1
timeout 1500 python tests/report_parity.py --out gpurun_out/parity_report.md > gpurun_out/parity_report.log 2>&1; tail -2 gpurun_out/parity_report.log
