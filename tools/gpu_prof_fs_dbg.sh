# ncu of the fast-scan kernel with RAIRS_FS_DBG bits set (timing experiments)
cfg=${1:-c4}; npb=${2:-2}; d=${3:-8}
RAIRS_FS_VARIANT=1 RAIRS_FS_DBG=$d timeout 300 python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/plain_dbg.log 2>&1 && \
RAIRS_FS_VARIANT=1 RAIRS_FS_DBG=$d timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs_scan -s 1 -c 1 -o gpurun_out/prof_fs_dbg$d python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/ncu_dbg.log 2>&1
tail -2 gpurun_out/ncu_dbg.log
