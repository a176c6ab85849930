for T in 65536 4096; do TOUCH_BYTES=$T timeout 300 python scripts/r2/buffers_probe.py; done
