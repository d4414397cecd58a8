# final default bench line (c4) + reference arm + launch list with the final code
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c4_reference.json 2> gpurun_out/bench_c4_ref.err; echo "ref rc=$?"
bash tools/gpu_bench_launches.sh; python tools/ncu_launches.py gpurun_out/launches_bench_c4.csv > gpurun_out/launches_summary.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
