# every measured path once on the final binary: bench lines under gpurun_out/final_*.json
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 900 python bench.py --steps 5 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/final_$out.json; python - "$out" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/final_{n}.json")); r=d["roofline"]
    print("%-22s %.3e  frac %.3f  e2e %.3e  iters %.2f  fer %.4f" % (n, d["value"], r["frac"], d["e2e"]["value"], d["config"]["mean_iters"], d["config"]["frame_error_rate"]))
except Exception as e: print(n, "ERR", open(f"gpurun_out/final_{n}.json").read()[:300])
PY
}
b C2 --no-cpu-baseline
b C3 --config C3 --no-cpu-baseline
b C4 --config C4 --frames 4096 --no-cpu-baseline
b C5 --config C5 --no-cpu-baseline
b C5p4 --config C5 --point 4 --no-cpu-baseline
b C2_direct --vn 1 --no-cpu-baseline
b C2_f16 --msg f16 --no-cpu-baseline
b C5_f16 --config C5 --msg f16 --no-cpu-baseline
b C2_pmf --input pmf --ebn0 0.5 --no-cpu-baseline
b C5_pmf --config C5 --input pmf --ebn0 3.5 --no-cpu-baseline
b C2_sym --symbol-out --no-cpu-baseline
b J3 --config J3 --no-cpu-baseline
b C2_logsp --algorithm logsp --no-cpu-baseline
