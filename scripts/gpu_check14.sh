cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python scripts/profile_integrator.py --steps 200 --grid 10 --P 132 > gpurun_out/prof_c14.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/cluster10 python scripts/profile_integrator.py --steps 200 --grid 10 --P 132 > gpurun_out/ncu_c10.log 2>&1
echo all done
