export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="8192 8192 16384 4096 4096 4096"
echo "default: $(PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
echo "ltpw7 tb15: $(DWT2_LARGE_TPW=7 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
echo "ltpw7 tb11: $(DWT2_LARGE_TPW=7 DWT2_TB_LARGE=11 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
echo "ltpw5 tb11: $(DWT2_LARGE_TPW=5 DWT2_TB_LARGE=11 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
echo "ltpw2 tb7: $(DWT2_LARGE_TPW=2 DWT2_TB_LARGE=7 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
echo "no-s3: $(DWT2_LARGE_S3=0 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py 16384 16384 16384 8192)"
