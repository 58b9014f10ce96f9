# Round evidence on the current binary, one gpurun call: GPU suite, smoke, default bench line (C4),
# reference arm, ncu launch list of the bench step, ncu --set full of the bench's lf_cluster launch.
# TAG names the outputs (gpurun_out/<TAG>_*).  Run each ncu pass only after its command exited 0 without ncu.
T=${TAG:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -30 gpurun_out/${T}_build.log; exit 1; }
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/${T}_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench.log 2>&1 && tail -1 gpurun_out/${T}_bench.log > gpurun_out/${T}_bench_default.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_reference.json
[ -n "$NO_NCU" ] && exit 0
timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_short.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:lf_cluster -s 3 -c 1 \
  -o gpurun_out/${T}_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/${T}_ncu_full.log; tail -3 gpurun_out/${T}_pytest_gpu.log; cat gpurun_out/${T}_smoke.log | tail -2; cat gpurun_out/${T}_bench_default.json
