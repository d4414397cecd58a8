# quick: scan-stage timing (c4 nprobe 2) + kernel time from the bench roofline
for i in 1 2; do timeout 300 python tools/time_fs.py c4 2 > gpurun_out/dbg.log 2>&1; echo "$(tail -1 gpurun_out/dbg.log)"; done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bq.json 2> gpurun_out/bq.err; echo "bench rc=$?"
python - <<'P'
import json; d=json.load(open('gpurun_out/bq.json')); r=d['roofline']
print(d['value'], d['recall10@10'], d['stage_ms_per_step'], r['avg_launch_ms'], r['frac'], r['stage_ms'])
P
