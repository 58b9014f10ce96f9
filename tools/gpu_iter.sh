# development GPU pass: parity tests + quick timings (args: pytest -k expression, optional)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu.log
for cfg in "C2 0 0 0 0,1" "C3 0 0 0 0,1" "C4 2048 0 0 0" "C5 16384 0 0 0" "C5 16384 0 4 0" "C1 0 0 0 0"; do
  timeout 300 python tools/quick_time.py $cfg 2>&1 | tail -3
done
