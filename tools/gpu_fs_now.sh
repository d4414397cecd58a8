# current fs_scan state: dbg sweep (stage timings) + one ncu --set full of fs_scan (c4, nprobe 2)
mkdir -p gpurun_out
for d in 0 8 32 40 1; do
RAIRS_FS_DBG=$d timeout 300 python tools/time_fs.py c4 2 > gpurun_out/dbg.log 2>&1
echo "dbg $d: $(tail -1 gpurun_out/dbg.log)"
done
bash tools/gpu_prof_fs.sh c4 2 > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/prof_fs_c4.ncu-rep fs_scan
