# tests + two short headline bench runs (value, stage split, frac)
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for i in 1 2; do python bench.py --compare-single 0 --updates 0 --no-cpu-baseline --latency-queries 0 --steps 20 2>&1 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['stage_ms_per_step'], d['roofline']['frac'])"; done
