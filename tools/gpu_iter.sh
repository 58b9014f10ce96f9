# development GPU pass: build, correctness smoke, quick timings (hard timeouts), parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
[ -z "${NODBG:-}" ] && timeout -s KILL 120 python tools/dbg_cluster.py 2>&1 | tail -8
echo "${QT:-C2 0 0 0 0;C3 0 0 0 0;C4 2048 0 0 0;C5 16384 0 0 0;C5 16384 0 4 0;C1 0 0 0 0}" | tr ';' '\n' | while read -r cfg; do
  timeout -s KILL 120 python tools/quick_time.py $cfg 2>&1 | tail -1
done
if [ -z "${NOTEST:-}" ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
  tail -6 gpurun_out/pytest_gpu.log
fi
