# scan-stage timing per kernel variant + parity subset + ncu of the default variant
for v in ${VARS:-0 1}; do RAIRS_FS_VARIANT=$v timeout 300 python tools/time_fs.py c4 2 > gpurun_out/dbg.log 2>&1; echo "var $v: $(tail -1 gpurun_out/dbg.log)"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q 2>&1 | tail -2
if [ -n "$PROF" ]; then bash tools/gpu_prof_fs.sh c4 2 > /dev/null 2>&1; python tools/ncu_brief.py gpurun_out/prof_fs_c4.ncu-rep fs_scan; fi
