# round-2 measurement: default bench line (c4), reference arm, c4 one-search DRAM traffic + launch list
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"; tail -2 gpurun_out/bench_ref.err
timeout 300 python tools/profile_step.py c4 2 auto 2 > gpurun_out/plain_c4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/ncu_traffic_c4_search.csv \
  python tools/profile_step.py c4 2 auto 2 > gpurun_out/ncu_traffic.log 2>&1
echo "ncu rc=$?"
