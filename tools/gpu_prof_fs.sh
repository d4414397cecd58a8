# ncu --set full of the query-major fast-scan kernel on one search (config, nprobe)
set -x
cfg=${1:-c4}; npb=${2:-2}
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/plain_$cfg.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs_scan -s 1 -c 1 -o gpurun_out/prof_fs_$cfg python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/ncu_fs_$cfg.log 2>&1
tail -3 gpurun_out/plain_$cfg.log
tail -3 gpurun_out/ncu_fs_$cfg.log
