# L2-policy experiment: the default build against NB_STCS=1 (W_e stored evict-first) and
# NB_STCS=2 (+ the decision's own-row copy with an L2 evict-first policy); alternating runs on one box.
# The variant libraries are built beforehand (NBLDPC_LIB / NBLDPC_DEFS, paper_1008_4370_b200/build.py).
L=paper_1008_4370_b200/lib
out=gpurun_out/r02f_l2hint.txt; : > $out
run() { # name lib defs args...
  n=$1; lib=$2; defs=$3; shift 3
  NBLDPC_LIB=$PWD/$L/$lib NBLDPC_DEFS="$defs" timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 > gpurun_out/l2hint_tmp.json
  python - "$n" "$*" <<'PY' | tee -a $out
import json,sys
try:
    d=json.load(open("gpurun_out/l2hint_tmp.json")); r=d["roofline"]
    print("%-8s %-22s %.4e  frac %.4f  ms/step %.2f  iters %.3f  FER %.5f  clk %s" % (sys.argv[1], sys.argv[2], d["value"], r["frac"], d["ms_per_step"], d["config"]["mean_iters"], d["config"]["frame_error_rate"], d["clocks"]["sm_mhz"]))
except Exception as e: print(sys.argv[1], "ERR", open("gpurun_out/l2hint_tmp.json").read()[:300])
PY
}
for rep in 1 2; do
  run base libnbldpc.so "" --config C4
  run stcs1 libnbldpc_stcs1.so "-DNB_STCS=1" --config C4
  run stcs2 libnbldpc_stcs2.so "-DNB_STCS=2" --config C4
done
for cfg in C3 C2; do
  run base libnbldpc.so "" --config $cfg
  run stcs1 libnbldpc_stcs1.so "-DNB_STCS=1" --config $cfg
  run stcs2 libnbldpc_stcs2.so "-DNB_STCS=2" --config $cfg
done
run base libnbldpc.so "" --config C5 --point 2
run stcs1 libnbldpc_stcs1.so "-DNB_STCS=1" --config C5 --point 2
rm -f gpurun_out/l2hint_tmp.json
