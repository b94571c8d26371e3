cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "
import paper_2405_00698_b200 as vx
ctx=vx.default_context()
print('fastmath', ctx.fastmath_check(1<<28, seed=777))
" > gpurun_out/abf_fastmath.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_configs.py tests/test_gpu_dump.py tests/test_gpu_parity.py -q -x > gpurun_out/abf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/abf_tests.log
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2 3; do
for v in main old; do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  echo -n "$v 10: " >> gpurun_out/abf_ab.txt; timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P 528 --steps 2000 2>&1 | tail -1 >> gpurun_out/abf_ab.txt
  echo -n "$v 6: " >> gpurun_out/abf_ab.txt; timeout -s KILL 120 python scripts/profile_integrator.py --grid 6 --P 256 --steps 5000 2>&1 | tail -1 >> gpurun_out/abf_ab.txt
  echo -n "$v 20: " >> gpurun_out/abf_ab.txt; timeout -s KILL 120 python scripts/profile_integrator.py --grid 20 --P 148 --steps 200 2>&1 | tail -1 >> gpurun_out/abf_ab.txt
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
cat gpurun_out/abf_fastmath.txt; tail -3 gpurun_out/abf_tests.log; cat gpurun_out/abf_ab.txt
