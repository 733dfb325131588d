# delta8 decode: GPU round-trip tests + C3 device time (tools/delta8_time.py)
make -C paper_2605_13928_b200/csrc -j16 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_delta.py -q -x 2>&1 | tail -1
for r in 1 2; do timeout 300 python tools/delta8_time.py 2>&1 | tail -1; done
