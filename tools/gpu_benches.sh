# round benches: c2pl headline (full line), top-100, c4, c5 (100M)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c2pl.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c2pl.log
timeout 300 python bench.py --k 100 --refine-factor 4 --no-cpu-baseline --compare-single 0 --updates 0 > gpurun_out/bench_top100.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --gt-queries 2000 --no-cpu-baseline --compare-single 0 > gpurun_out/bench_c4.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c4.log
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --gt-queries 500 --nprobe 64 --no-cpu-baseline --compare-single 0 > gpurun_out/bench_c5.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c5.log
echo done
