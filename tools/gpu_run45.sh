set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --gt-queries 200 --nprobe 64 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c5.log
echo done
