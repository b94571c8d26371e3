cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for rep in 1 2; do
for r in 3 4 5 6 8; do
echo -n "ratio=$r: " >> gpurun_out/ratio.txt
VX_FILLER_RATIO=$r timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 5000 >> gpurun_out/ratio.txt 2>&1
done; done
echo -n "filler off: " >> gpurun_out/ratio.txt
VX_FILLER=0 timeout 300 python scripts/profile_integrator.py --grid 10 --P 2867 --steps 5000 >> gpurun_out/ratio.txt 2>&1
cat gpurun_out/ratio.txt
timeout 900 python bench.py > gpurun_out/bench_fill.log 2> gpurun_out/bench_fill.err; tail -1 gpurun_out/bench_fill.log | cut -c1-600
