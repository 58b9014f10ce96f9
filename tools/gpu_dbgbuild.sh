# bounds-checked build (device asserts) running the GPU parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
NBLDPC_LIB=/tmp/nbl_dbg/libnbldpc.so NBLDPC_DEFS="-DNB_BOUNDS_CHECK" python -c "import sys; sys.path.insert(0,'.'); from paper_1008_4370_b200 import build; build.build(force=True)" || exit 1
NBLDPC_LIB=/tmp/nbl_dbg/libnbldpc.so timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_bounds.log 2>&1; echo "bounds-checked pytest exit $?"; tail -3 gpurun_out/pytest_gpu_bounds.log
