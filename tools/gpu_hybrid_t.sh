# hybrid SEIL layout: tiny-cell threshold sweep on c4 / c4pl / c2pl
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seil_paper.py -x -q > gpurun_out/hyb_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hyb_tests.log
for T in 4 8 16 32; do for c in c4 c4pl c2pl; do
  RAIRS_SEIL_TINY=$T timeout 900 python bench.py --config $c --seil-layout hybrid --steps 10 --warmup 3 --gt-queries 1000 --no-cpu-baseline --compare-single 0 \
     --latency-queries 0 --k1 0 --updates 0 > gpurun_out/hyb_$c.json 2> gpurun_out/hyb_$c.err; echo -n "T=$T rc=$? "
  python - $c <<'P'
import json,sys; d=json.load(open(f'gpurun_out/hyb_{sys.argv[1]}.json')); s=d['seil_layouts']
print(sys.argv[1], d['value'], {k:(v['qps'],v['dco_per_query']) for k,v in s.items() if isinstance(v,dict)})
P
done; done
