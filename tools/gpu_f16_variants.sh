# build the F16 storage variants and compare FER / speed (tools/dbg_f16.py)
for v in "half:" "fixed:-DNB_MSG16_FIXED"; do
  name=${v%%:*}; defs=${v#*:}
  NBLDPC_LIB=/tmp/nbl_$name/libnbldpc.so NBLDPC_DEFS="$defs" python -c "import sys; sys.path.insert(0,'.'); from paper_1008_4370_b200 import build; build.build(force=True)" > /tmp/b_$name.log 2>&1 || { tail -20 /tmp/b_$name.log; exit 1; }
  echo "== $name"; NBLDPC_LIB=/tmp/nbl_$name/libnbldpc.so timeout -s KILL 600 python tools/dbg_f16.py
done
