set -x
mkdir -p gpurun_out
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 200 python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lut_|lm_|refine|coarse|probe" -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py c2pl 4 auto 3 > gpurun_out/ncu_launch.log 2>&1
timeout 200 python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"coarse_topw|coarse_certify|lm_tensor|lm_select|refine_stage|lut_tiles" -s 52 -c 6 -o gpurun_out/prof_final python tools/profile_step.py c2pl 4 auto 1 > gpurun_out/ncu_full.log 2>&1
echo done
