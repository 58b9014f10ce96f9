# every measured path once on the current binary (round 2): bench lines under gpurun_out/final_*.json and a
# one-line summary each in gpurun_out/final_matrix.txt.  The default bench line is C4 (BASELINE configs[3]).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 1200 python bench.py --steps 5 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/final_$out.json; python - "$out" <<'PY' | tee -a gpurun_out/final_matrix.txt
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/final_{n}.json")); r=d["roofline"]; c=d["config"]
    print("%-14s %.3e  frac %.3f  e2e %.3e  iters %5.2f  FER %.5f  BER %.2e  undet %d  ms/step %.1f" % (n, d["value"], r["frac"], d.get("e2e", {}).get("value", 0), c["mean_iters"], c["frame_error_rate"], c.get("bit_error_rate", 0), c.get("undetected_frames", 0), d["ms_per_step"]))
except Exception as e: print(n, "ERR", open(f"gpurun_out/final_{n}.json").read()[:300])
PY
}
: > gpurun_out/final_matrix.txt
b C4 ${C4ARGS:-}
b C2 --config C2 --no-cpu-baseline
b C3 --config C3 --no-cpu-baseline
for p in 0 1 2 3 4; do b C5p$p --config C5 --point $p --no-cpu-baseline; done
b C1 --config C1 --no-cpu-baseline --no-e2e
[ -n "$QUICK" ] && exit 0
b C2_direct --config C2 --vn 1 --no-cpu-baseline
b C2_f16 --config C2 --msg f16 --no-cpu-baseline
b C4_f16 --config C4 --msg f16 --no-cpu-baseline
b C5_f16 --config C5 --point 3 --msg f16 --no-cpu-baseline
b C2_pmf --config C2 --input pmf --ebn0 0.5 --no-cpu-baseline
b C5_pmf --config C5 --input pmf --ebn0 3.5 --no-cpu-baseline
b C2_sym --config C2 --symbol-out --no-cpu-baseline
b J3 --config J3 --no-cpu-baseline
b C2_logsp --config C2 --algorithm logsp --no-cpu-baseline
