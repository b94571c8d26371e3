cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out; rm -f gpurun_out/ratio2.txt
for rep in 1 2; do
for r in 4 6 8 10 14; do
echo -n "ratio=$r: " >> gpurun_out/ratio2.txt
VX_FILLER_RATIO=$r timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 5000 2>&1 | tail -1 >> gpurun_out/ratio2.txt
done; done
echo -n "filler off: " >> gpurun_out/ratio2.txt
VX_FILLER=0 timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 5000 2>&1 | tail -1 >> gpurun_out/ratio2.txt
cat gpurun_out/ratio2.txt
