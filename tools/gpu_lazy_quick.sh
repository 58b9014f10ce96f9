# quick check of the lazy decision: C4 / C3 bench lines, then the q = 256 parity, stress and shard tests
for cfg in C4 C3; do
  timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config $cfg 2>&1 | tail -1 > gpurun_out/lazy_$cfg.json
  python - $cfg <<'PY'
import json,sys
try:
    d=json.load(open(f"gpurun_out/lazy_{sys.argv[1]}.json")); print(sys.argv[1], "%.4e frac %.4f ms %.2f iters %.4f FER %.6f undet %d clk %s" % (d["value"], d["roofline"]["frac"], d["ms_per_step"], d["config"]["mean_iters"], d["config"]["frame_error_rate"], d["config"]["undetected_frames"], d["clocks"]["sm_mhz"]))
except Exception as e: print("ERR", open(f"gpurun_out/lazy_{sys.argv[1]}.json").read()[-600:])
PY
done
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_shard.py -m gpu -x -q -k "C3 or C4 or invariance or largest or stress or repeat or shard or strong or host or edge" > gpurun_out/lazy_pytest.log 2>&1; tail -15 gpurun_out/lazy_pytest.log
