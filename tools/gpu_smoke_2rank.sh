# __graft_entry__ smoke on the GPU + the 2-rank sharded bench path run functionally on one GPU (gloo)
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
RAIRS_BENCH_BACKEND=gloo RAIRS_BENCH_ONE_GPU=1 timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 --compare-single 0 --updates 0 --latency-queries 0 --k1 0 --seil-paper 0 --no-cpu-baseline > gpurun_out/bench_c4_2rank.json 2> gpurun_out/bench_c4_2rank.err; echo "2rank rc=$?"; tail -2 gpurun_out/bench_c4_2rank.err
