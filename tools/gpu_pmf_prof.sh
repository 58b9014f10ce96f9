# section 8(f) row 1 evidence: bench lines (pmf input, symbol outputs) + one ncu --set full of the pmf cluster kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
b() { out=$1; shift; timeout -s KILL 600 python bench.py --steps 5 --warmup 3 "$@" 2>&1 | tail -1 > gpurun_out/$out.json; echo "$out: $(cut -c1-160 gpurun_out/$out.json)"; }
b r01_bench_C2_pmf --input pmf --ebn0 0.5 --cpu-frames 16
b r01_bench_C3_pmf --config C3 --input pmf --ebn0 1.0 --cpu-frames 4
b r01_bench_C5_pmf --config C5 --point 3 --input pmf --ebn0 3.5 --cpu-frames 64
b r01_bench_C2_symbol_out --symbol-out --cpu-frames 16
b r01_bench_C2_pmf_symbol_out --input pmf --ebn0 0.5 --symbol-out --cpu-frames 8
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --input pmf --ebn0 0.5"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lf_cluster -s 3 -c 1 -o gpurun_out/pmf_full $B > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
