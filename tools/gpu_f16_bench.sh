# section 8(f) row 4 evidence: F16-message bench lines + one ncu --set full of the C2 F16 kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 900 python bench.py --steps 5 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/$out.json; python - "$out" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/{n}.json")); r=d["roofline"]
    print(n, "%.3e" % d["value"], "%.1f ms" % d["ms_per_step"], "iters %.2f" % d["config"]["mean_iters"], r["bound"], "frac %.3f" % r["frac"], "fer %.4f" % d["config"]["frame_error_rate"], "e2e %.3e" % d["e2e"]["value"])
except Exception as e: print(n, "ERR", open(f"gpurun_out/{n}.json").read()[:300])
PY
}
b r01_bench_C2_f16 --msg f16 --no-cpu-baseline
b r01_bench_C3_f16 --config C3 --msg f16 --no-cpu-baseline
b r01_bench_C5_f16 --config C5 --msg f16 --no-cpu-baseline
b r01_bench_C5p3_f16 --config C5 --point 3 --msg f16 --no-cpu-baseline
b r01_bench_C5p3_f32 --config C5 --point 3 --no-cpu-baseline
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --msg f16"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lf_cluster -s 3 -c 1 -o gpurun_out/c2_f16_full $B > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
