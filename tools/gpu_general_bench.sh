# section 8(f) row 3 evidence: the general-column-weight kernel on J3 ((3,6), GF(64)) and on C2 / C5 for comparison
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 900 python bench.py --steps 3 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/$out.json; python - "$out" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/{n}.json")); r=d["roofline"]
    print(n, "%.3e" % d["value"], "%.1f ms" % d["ms_per_step"], "iters %.2f" % d["config"]["mean_iters"], r["bound"], r.get("pipe"), "frac %.3f" % r["frac"], "fer %.3f" % d["config"]["frame_error_rate"], "e2e %.3e" % d["e2e"]["value"], "cpu %.3e" % d.get("cpu_baseline", {}).get("value", 0))
except Exception as e: print(n, "ERR", open(f"gpurun_out/{n}.json").read()[:300])
PY
}
b r01_bench_J3_general --config J3 --cpu-frames 4
b r01_bench_C2_general --vn 2 --cpu-frames 4
b r01_bench_C5_general --config C5 --point 4 --frames 8192 --vn 2 --cpu-frames 16
B="python bench.py --config J3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lfg_frame -s 3 -c 1 -o gpurun_out/j3_full $B > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
