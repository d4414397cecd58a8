set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1
for dg in 0 31; do
  RAIRS_LM_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lm_tensor|coarse" -c 60 --csv --log-file gpurun_out/diag3_$dg.csv python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_diag3_$dg.log 2>&1
done
timeout 300 python -m pytest tests -m gpu -x -q -k "search_parity or many_queries or full_size_sampled" > gpurun_out/gpu_tests_a.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_a.log
echo done
