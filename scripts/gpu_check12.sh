cd $GRAFT_REPO_ROOT
timeout 300 python scripts/profile_integrator.py --steps 100 --grid 10 --P 148 > gpurun_out/prof_s10.log 2>&1 && \
timeout 300 python scripts/profile_integrator.py --steps 30 --grid 20 --P 148 > gpurun_out/prof_s20.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 -o gpurun_out/stream10 python scripts/profile_integrator.py --steps 100 --grid 10 --P 148 > gpurun_out/ncu_s10.log 2>&1
echo all done
