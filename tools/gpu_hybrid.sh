# hybrid SEIL layout: parity + the three layouts on c4 / c4pl / c2pl
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seil_paper.py -x -q > gpurun_out/hyb_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/hyb_tests.log
for c in c4 c4pl c2pl; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --gt-queries 1000 --no-cpu-baseline --compare-single 0 \
     --latency-queries 0 --k1 0 --updates 0 > gpurun_out/hyb_$c.json 2> gpurun_out/hyb_$c.err; echo "$c rc=$?"
  python - $c <<'P'
import json,sys; d=json.load(open(f'gpurun_out/hyb_{sys.argv[1]}.json')); s=d['seil_layouts']
print(sys.argv[1], d['value'], {k:(v['qps'],v['dco_per_query']) for k,v in s.items() if isinstance(v,dict)})
P
done
