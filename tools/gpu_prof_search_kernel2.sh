# ncu --set full of one kernel (regex) inside the NVTX range 'search' of tools/profile_step.py:
#   bash tools/gpu_prof_search_kernel2.sh <cfg> <nprobe> <regex> <name>
cfg=$1; npb=$2; rx=$3; nm=$4
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/plain_$nm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "search/" -k regex:$rx -c 1 -o gpurun_out/prof_$nm python tools/profile_step.py $cfg $npb auto 2 > gpurun_out/ncu_$nm.log 2>&1
tail -1 gpurun_out/ncu_$nm.log
