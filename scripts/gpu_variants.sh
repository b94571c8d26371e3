# A/B the integrator variants built under _variants/<name> (development aid):
# a bit-exactness check and two timing reps per variant.
cd $GRAFT_REPO_ROOT
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v check: "; timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "lattice_integrator_bit_exact or large" ${VARIANT_TESTS} 2>&1 | tail -1
done
for rep in 1 2; do
for v in $(ls _variants); do
  cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
  echo -n "$v: "; timeout -s KILL 120 python scripts/profile_integrator.py --steps 5000 ${VARIANT_ARGS} 2>&1 | tail -1
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
