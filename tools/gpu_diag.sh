# lm_tensor bottleneck isolation (timing only; results are wrong with RAIRS_LM_DIAG != 0)
set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/plain.log 2>&1
for dg in 0 1 2 4 3 7; do
  RAIRS_LM_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lm_tensor|coarse_topw|coarse_certify" -c 60 --csv --log-file gpurun_out/diag_$dg.csv python tools/profile_step.py c2pl 4 auto 2 > gpurun_out/ncu_diag_$dg.log 2>&1
done
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --gt-queries 200 --nprobe 64 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c5.log
echo done
