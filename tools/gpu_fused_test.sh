RAIRS_LM_FUSED=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -k "listmajor or massive or stats or overlapped or c2pl" 2>&1 | tail -4
for f in 0 1; do RAIRS_LM_FUSED=$f SCAN_MODE=listmajor python tools/time_fs.py c2pl 4 10 2>&1 | tail -1; done
