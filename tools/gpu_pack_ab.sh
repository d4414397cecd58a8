# packed-pair fast scan A/B: GPU suite, c4 bench with and without RAIRS_FS_PACK
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
for pk in 0 1; do
RAIRS_FS_PACK=$pk timeout 600 python bench.py --steps 10 --warmup 3 --compare-single 0 --no-cpu-baseline > gpurun_out/bench_pk$pk.json 2> gpurun_out/bench_pk$pk.err; echo "pk$pk rc=$?"
done
python - <<'PY'
import json
for pk in (0,1):
    d=json.loads(open(f'gpurun_out/bench_pk{pk}.json').read().strip().split('\n')[-1])
    print(pk, d['value'], d['ms_per_step'], d['stage_ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['k1'])
PY
