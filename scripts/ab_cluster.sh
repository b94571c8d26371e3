# A/B of the cluster integrator variants under _variants/ (10^3, P=528, 2000 steps)
cd $GRAFT_REPO_ROOT
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v check: "; timeout -s KILL 300 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_configs.py -q -x -k "cluster or 10 or 8" 2>&1 | tail -1
done
for rep in 1 2 3; do
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v: "; timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P 528 --steps 2000 2>&1 | tail -1
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
