python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -k "simt or massive or c4_full or stats" 2>&1 | tail -1
for d in 1 0; do RAIRS_FS_DEFER=$d python tools/time_fs.py c4 2 10 2>&1 | tail -1 | sed "s/^/defer $d: /"; done
RAIRS_FS_DEFER=1 python tools/time_fs.py c4pl 3 10 2>&1 | tail -1
