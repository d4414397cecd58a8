# final lines of the non-default configs with the final code
mkdir -p gpurun_out
python bench.py --config c2pl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2pl.json 2> gpurun_out/bench_c2pl.err; echo "c2pl rc=$?"
python bench.py --config c3pl --steps 5 --warmup 3 --gt-queries 1000 --latency-queries 50 --no-cpu-baseline > gpurun_out/bench_c3pl.json 2> gpurun_out/bench_c3pl.err; echo "c3pl rc=$?"
python bench.py --config c5pl --steps 5 --warmup 3 --gt-queries 1000 --compare-single 0 --latency-queries 50 --no-cpu-baseline > gpurun_out/bench_c5pl.json 2> gpurun_out/bench_c5pl.err; echo "c5pl rc=$?"
python bench.py --config c5 --nprobe 64 --steps 5 --warmup 3 --compare-single 0 --updates 0 --gt-queries 1000 --latency-queries 50 --k1 0 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
