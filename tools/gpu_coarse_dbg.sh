for d in 0 1; do
COARSE_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/cd_$d.csv python tools/profile_step.py c4 2 auto 2 > /dev/null 2>&1
grep -E "coarse_topw|coarse_certify|probe_" gpurun_out/cd_$d.csv | awk -F'","' '{print "dbg '$d'", $7, $NF}' | cut -c1-120
done
