# pmf tests + pmf bench lines (section 8(f) row 1)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests/test_gpu_pmf.py -q -x 2>&1 | tail -2
for a in "--input pmf --ebn0 0.5" "--input pmf --ebn0 0.5 --symbol-out" "--config C5 --point 3 --input pmf --ebn0 3.5" "--config C3 --input pmf --ebn0 1.0" ${EXTRA:-}; do
  echo "== $a"
  timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --cpu-frames 8 $a 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
    d=json.loads(l); r=d['roofline']
    print('%.3e' % d['value'], '%.2f ms' % d['ms_per_step'], 'iters %.2f' % d['config']['mean_iters'], r['bound'], r.get('pipe'), 'frac %.3f' % r['frac'], 'e2e %.3e' % d['e2e']['value'])
except Exception: print(l[:400])
"
done
