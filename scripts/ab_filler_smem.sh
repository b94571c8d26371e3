# A/B: the filler with shared-memory state (in-tree build) against _variants/*
# (P = 2867 10^3, 5000 steps), filler parity tests first; then the plan-wait
# trace at P = 256 x world (6^3) and the config-3 bench
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-fsm}
timeout -s KILL 600 python -m pytest tests/test_gpu_filler.py tests/test_gpu_cluster.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2; do
for v in main $(ls _variants 2>/dev/null); do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  echo -n "$v: " >> gpurun_out/${T}_ab.txt; VX_FILLER_STATS=${STATS:-0} timeout -s KILL 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 5000 2>&1 | tail -2 | tr '\n' ' ' >> gpurun_out/${T}_ab.txt; echo >> gpurun_out/${T}_ab.txt
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
VX_EVO_TRACE=1 timeout -s KILL 600 python scripts/plan_time.py > gpurun_out/${T}_plan.txt 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err
tail -3 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_ab.txt; cat gpurun_out/${T}_plan.txt; tail -1 gpurun_out/${T}_bench.log | cut -c1-300
