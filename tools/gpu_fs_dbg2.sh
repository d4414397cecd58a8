for v in ${VARS:-0 1 2}; do for d in ${DBGS:-0 8}; do
RAIRS_FS_VARIANT=$v RAIRS_FS_DBG=$d python tools/time_fs.py ${CFG:-c4} ${NPB:-2} > gpurun_out/dbg.log 2>&1
echo "var $v dbg $d: $(tail -1 gpurun_out/dbg.log)"
done; done
