# ncu --set full of the pass kernel on C2 (host-driven loop so kernels are profilable)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/quick_time.py ${CFG:-C2} ${FR:-1024} 0 ${PT:-0} ${VN:-0} -1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nb_pass -s ${SKIP:-40} -c ${CNT:-2} -o gpurun_out/${OUT:-prof_c2} $CMD > gpurun_out/prof_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/prof_ncu.log; cat gpurun_out/prof_plain.log
