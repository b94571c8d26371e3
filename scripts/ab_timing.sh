cd ${GRAFT_REPO_ROOT:-.}
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2 3; do
for v in main $(ls _variants); do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  echo -n "$v: "; timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P 528 --steps 2000 2>&1 | tail -1
  echo -n "$v nofill: "; VX_FILLER=0 timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P 528 --steps 2000 2>&1 | tail -1
done; done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
