# The bulk-copy-fed streaming kernel (default) against the L1-fed one
# (VX_STREAM_TMA=0) and the _variants/* builds (stage-ring depths): 20^3
# parity tests on the in-tree build, then timing reps.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_dump.py tests/test_gpu_parity.py -q -x -k "20 or stream" 2>&1 | tail -2
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2 3; do
  for v in main legacy $(ls _variants 2>/dev/null); do
    case $v in main|legacy) cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so;; *) cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so;; esac
    m=1; [ $v = legacy ] && m=0
    echo -n "$v: "; VX_STREAM_TMA=$m timeout -s KILL 120 python scripts/profile_integrator.py --grid 20 --P ${P:-148} --steps ${STEPS:-200} 2>&1 | tail -1
  done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
