# per-kernel device times of one search (NVTX "search" range): <cfg> <nprobe> <scan> [env...]
cfg=$1; npb=$2; sm=$3; tag=$4
timeout 300 python tools/profile_step.py $cfg $npb $sm 2 > gpurun_out/plain_l_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/launch_$tag.csv python tools/profile_step.py $cfg $npb $sm 2 > /dev/null 2>&1
python3 tools/traffic_from_ncu.py gpurun_out/launch_$tag.csv $cfg gpurun_out/traffic_$tag.json 1 $sm $npb > /dev/null
python3 -c "
import json; d=json.load(open('gpurun_out/traffic_$tag.json'))
for k,v in d['kernels'].items(): print('$tag', k, round(v['duration_per_search_ns']/1e3,1), 'us', round(v['dram_bytes_per_search']/1e6,1), 'MB', v['launches'])"
