# A/B of the cluster integrator: the in-tree build against every _variants/*
# build (10^3, P=528, 2000 steps), after the cluster parity tests on the in-tree build
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-ab}
timeout -s KILL 600 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_configs.py tests/test_gpu_dump.py tests/test_gpu_filler.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2 3; do
for v in main $(ls _variants 2>/dev/null); do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  echo -n "$v: " >> gpurun_out/${T}_ab.txt; timeout -s KILL 120 python scripts/profile_integrator.py --grid ${GRID:-10} --P ${P:-528} --steps ${STEPS:-2000} 2>&1 | tail -1 >> gpurun_out/${T}_ab.txt
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
tail -5 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_ab.txt
