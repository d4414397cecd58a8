# time the fast-scan kernel with parts disabled (RAIRS_FS_DBG bits; results are wrong, timing only)
for d in ${DBGS:-0 1 2 4 7}; do
RAIRS_FS_VARIANT=1 RAIRS_FS_DBG=$d python tools/time_fs.py c4 2 > gpurun_out/dbg_$d.log 2>&1
echo "dbg $d: $(tail -1 gpurun_out/dbg_$d.log)"
done
