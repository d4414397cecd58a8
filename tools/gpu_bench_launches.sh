# ncu launch list (gpu__time_duration, cold-cache, serialised) of the default bench command with the side lines off
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --compare-single 0 --updates 0 --latency-queries 0 --k1 0 --seil-paper 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv --log-file gpurun_out/launches_bench_c4.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_bench.log
