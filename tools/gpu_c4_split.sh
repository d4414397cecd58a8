for sp in 0 4 8 16; do
RAIRS_COARSE_SPLIT=$sp timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --gt-queries 1000 --no-cpu-baseline --compare-single 0 --latency-queries 0 --updates 0 2>&1 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($sp, d['value'], d['stage_ms_per_step'], d['recall10@10'])"
done
