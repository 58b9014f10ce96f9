# probe-count sweep of the lazy decision: NB_PROBE_SHIFT = 3 (default: nch / 8 probe chunks per CTA and pass), 2, 1
L=paper_1008_4370_b200/lib
out=gpurun_out/r02g_probe_sweep.txt; : > $out
run() { n=$1; lib=$2; defs=$3; shift 3
  NBLDPC_LIB=$PWD/$L/$lib NBLDPC_DEFS="$defs" timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 > gpurun_out/ps_tmp.json
  python - "$n" "$*" <<'PY' | tee -a $out
import json,sys
try:
    d=json.load(open("gpurun_out/ps_tmp.json")); r=d["roofline"]
    print("%-8s %-22s %.4e  frac %.4f  ms/step %.2f  iters %.6f  FER %.6f  clk %s" % (sys.argv[1], sys.argv[2], d["value"], r["frac"], d["ms_per_step"], d["config"]["mean_iters"], d["config"]["frame_error_rate"], d["clocks"]["sm_mhz"]))
except Exception as e: print(sys.argv[1], "ERR", open("gpurun_out/ps_tmp.json").read()[-300:])
PY
}
for cfg in C4 C3; do
  run shift3 libnbldpc.so "" --config $cfg
  run shift1 libnbldpc_ps1.so "-DNB_PROBE_SHIFT=1" --config $cfg
done
rm -f gpurun_out/ps_tmp.json
