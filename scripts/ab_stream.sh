cd $GRAFT_REPO_ROOT
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v check: "; timeout -s KILL 300 python -m pytest tests/test_gpu_configs.py -q -x -k "20" 2>&1 | tail -1
done
for rep in 1 2 3; do
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v: "; timeout -s KILL 120 python scripts/profile_integrator.py --grid 20 --P 148 --steps 200 2>&1 | tail -1
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
