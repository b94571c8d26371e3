cd $GRAFT_REPO_ROOT
for g in 10 8 7; do
timeout -s KILL 300 python scripts/profile_integrator.py --steps 2000 --grid $g --P 528 > gpurun_out/p22_c$g.log 2>&1
VX_INTEGRATOR=stream timeout -s KILL 300 python scripts/profile_integrator.py --steps 2000 --grid $g --P 528 > gpurun_out/p22_s$g.log 2>&1
done
cat gpurun_out/p22_*.log
