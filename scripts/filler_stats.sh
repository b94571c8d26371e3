# filler development aid: parity tests, then who integrated what and when
# (VX_FILLER_STATS=1), and throughput with / without the filler
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
T=${TAG:-fs}
timeout -s KILL 600 python -m pytest tests/test_gpu_filler.py tests/test_gpu_cluster.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for c in 16 8; do
VX_FILLER_STATS=1 VX_FILLER=1 VX_FILLER_CTAS=$c timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 2000 >> gpurun_out/${T}.txt 2>&1
done
VX_FILLER_STATS=1 VX_FILLER=2 timeout 300 python scripts/profile_integrator.py --grid 10 --P 64 --steps 2000 >> gpurun_out/${T}.txt 2>&1
for rep in 1 2; do
for f in 0 1; do
echo -n "VX_FILLER=$f: " >> gpurun_out/${T}.txt
VX_FILLER=$f timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 2000 >> gpurun_out/${T}.txt 2>&1
done; done
cat gpurun_out/${T}.txt
