set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "fallback_split or coarse or full_size_sampled" > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 400 python tools/profile_c5_coarse.py > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"coarse|probe_" -c 200 --csv --log-file gpurun_out/launches_c5.csv python tools/profile_c5_coarse.py > gpurun_out/ncu_c5.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
echo done
