for nb in 8 16 32 48 64; do echo "bands $nb"; DWT2_HOST_BANDS=$nb timeout 300 python scripts/e2e_probe.py 2>&1 | tail -4; done
