# coarse stage on c4: ncu full capture of coarse_topw + certify, and dbg split timings
mkdir -p gpurun_out
bash tools/gpu_prof_kernel.sh c4 2 coarse_topw coarse_c4
bash tools/gpu_prof_kernel.sh c4 2 coarse_certify certify_c4
for d in 0 1; do
COARSE_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/cd_$d.csv python tools/profile_step.py c4 2 auto 2 > /dev/null 2>&1
grep -E "coarse_topw|coarse_certify|probe_" gpurun_out/cd_$d.csv | awk -F'","' '{print "dbg '$d'", $7, $NF}' | cut -c1-120
done
