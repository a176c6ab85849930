export DWT2_LIB=build/variants/libdwt2_tuning.so
for mt in 16 8 4; do echo "MINTB $mt"; DWT2_K2_MINTB=$mt timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8; done
for mt in 16 8 4; do echo "INV MINTB $mt"; DWT2_K2INV_MINTB=$mt timeout 300 python scripts/inverse_bench.py 2>&1 | grep -i "97\|k2" | head -5; done
