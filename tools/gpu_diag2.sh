set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1
for dg in 0 7 15 23 31; do
  RAIRS_LM_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lm_tensor" -c 6 --csv --log-file gpurun_out/diag2_$dg.csv python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_diag2_$dg.log 2>&1
done
echo done
