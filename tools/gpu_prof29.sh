set -x
mkdir -p gpurun_out
timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lm_select|refine_stage|coarse_topw|coarse_certify" -s 52 -c 4 -o gpurun_out/prof_lm8 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/ncu_full.log 2>&1
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --gt-queries 200 --nprobe 64 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c5.log
echo done
