mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -5
