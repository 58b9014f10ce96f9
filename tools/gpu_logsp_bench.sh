# section 8(f) row 2 evidence: conventional Log-SP bench lines next to the Log-Fourier ones (same workloads)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 900 python bench.py --steps 3 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/$out.json; python - "$out" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/{n}.json")); r=d["roofline"]
    print(n, "%.3e" % d["value"], "%.1f ms" % d["ms_per_step"], "iters %.2f" % d["config"]["mean_iters"], r["bound"], r.get("pipe"), "frac %.3f" % r["frac"], "fer %.3f" % d["config"]["frame_error_rate"], "cpu %.3e" % d.get("cpu_baseline", {}).get("value", 0))
except Exception as e: print(n, "ERR", open(f"gpurun_out/{n}.json").read()[:300])
PY
}
b r01_bench_C2_logsp --algorithm logsp --cpu-frames 4
b r01_bench_C5_logsp --config C5 --point 4 --algorithm logsp --frames 8192 --cpu-frames 8
b r01_bench_C5_lf_p4 --config C5 --point 4 --frames 8192 --cpu-frames 64
b r01_bench_C3_logsp --config C3 --algorithm logsp --frames 1024 --cpu-frames 2
b r01_bench_C4_logsp --config C4 --algorithm logsp --frames 256 --no-cpu-baseline
