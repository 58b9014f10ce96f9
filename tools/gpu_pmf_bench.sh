# bench lines of the symbol-pmf input and the symbol outputs (section 8(f) row 1), plus the LLR baselines
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() { echo "== $*"; timeout -s KILL 600 python bench.py "$@" 2>&1 | tail -1; }
run --steps 5 --warmup 3
run --steps 5 --warmup 3 --vn 1 --cpu-frames 16
run --steps 5 --warmup 3 --symbol-out --cpu-frames 16
run --steps 5 --warmup 3 --input pmf --ebn0 0.5 --cpu-frames 8
run --steps 5 --warmup 3 --input pmf --ebn0 0.5 --symbol-out --cpu-frames 8
run --config C5 --point 3 --steps 5 --warmup 3 --input pmf --ebn0 3.5 --cpu-frames 64
