# A/B timing of one build under an environment switch: AB_ENV="NAME=value"
for cfg in "C2 0 0 0 0" "C3 0 0 0 0" "C4 2048 0 0 0" "C5 16384 0 0 0" "C5 16384 0 4 0"; do
  a=$(timeout -s KILL 120 python tools/quick_time.py $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f' % d['ns_per_frame_iter'])")
  b=$(env ${AB_ENV} timeout -s KILL 120 python tools/quick_time.py $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f' % d['ns_per_frame_iter'])")
  echo "$cfg  default ${a} ns  |  ${AB_ENV}: ${b} ns"
done
