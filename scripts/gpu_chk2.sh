mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -3
timeout 300 python scripts/sanitize_driver.py
for t in memcheck racecheck synccheck; do
  /usr/bin/time -f "$t %e s" timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san_$t.log
done
