# build variants and time them: VARIANTS="name:defs ..." ; CSL="cluster sizes" ; QT="cfg args;cfg args"
for v in ${VARIANTS:-"m2:-DNB_CLUSTER_MINB=2" "m3:-DNB_CLUSTER_MINB=3"}; do
  name=${v%%:*}; defs=${v#*:}
  NBLDPC_LIB=/tmp/nbl_$name/libnbldpc.so NBLDPC_DEFS="$defs" python -c "import sys; sys.path.insert(0,'.'); from paper_1008_4370_b200 import build; build.build(force=True)" || exit 1
  for cs in ${CSL:-2}; do
    echo "${QT:-C2 0 0 0 0}" | tr ';' '\n' | while read -r cfg; do
      echo "variant $name cs=$cs cfg=$cfg"
      NBLDPC_LIB=/tmp/nbl_$name/libnbldpc.so NBLDPC_CLUSTER_SIZE=$cs timeout -s KILL 120 python tools/quick_time.py $cfg 2>&1 | tail -1
    done
  done
done
