# A/B of the cluster integrator timing only (no tests), with and without the
# one-SM filler: in-tree build vs every _variants/* build (10^3, P, steps)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2 3 4; do
for v in main $(ls _variants 2>/dev/null); do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  for f in 1 0; do
  echo -n "$v filler=$f: "; VX_FILLER=$f timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P ${P:-528} --steps ${STEPS:-2000} 2>&1 | tail -1
  done
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
