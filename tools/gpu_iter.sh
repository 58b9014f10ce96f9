# development GPU pass: build, quick timings (each under a hard timeout), parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for cfg in ${QT:-"C1 0 0 0 0" "C2 512 0 0 0" "C2 0 0 0 0,1" "C3 0 0 0 0" "C4 2048 0 0 0" "C5 16384 0 0 0" "C5 16384 0 4 0"}; do
  timeout -s KILL 120 python tools/quick_time.py $cfg 2>&1 | tail -2
done
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest_gpu.log
