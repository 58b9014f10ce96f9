# ncu --set full of one kernel: CFG FR PT VN GR KREGEX SKIP CNT OUT env vars
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/quick_time.py ${CFG:-C2} ${FR:-512} 0 ${PT:-0} ${VN:-0} ${GR:-0}"
timeout -s KILL 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-lf_cluster} -s ${SKIP:-2} -c ${CNT:-1} -o gpurun_out/${OUT:-prof_c2} $CMD > gpurun_out/prof_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/prof_ncu.log; cat gpurun_out/prof_plain.log
