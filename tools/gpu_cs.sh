# cluster-size sweep on the bench workload with DRAM traffic (ncu metrics pass)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for cs in ${CSL:-2 4}; do
  echo "cs=$cs"
  NBLDPC_CLUSTER_SIZE=$cs timeout -s KILL 120 python tools/quick_time.py ${CFG:-C2} ${FR:-0} 0 ${PT:-0} 2>&1 | tail -1
  NBLDPC_CLUSTER_SIZE=$cs timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lf_cluster -s 1 -c 1 python tools/quick_time.py ${CFG:-C2} ${FR:-0} 0 ${PT:-0} 2>&1 | grep -E "dram__|gpu__time"
done
