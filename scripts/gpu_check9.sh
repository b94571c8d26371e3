cd $GRAFT_REPO_ROOT
timeout 300 python scripts/profile_integrator.py --steps 2000 > gpurun_out/prof_plain.log 2>&1
VX_LATTICE_WAVE=0 timeout 300 python scripts/profile_integrator.py --steps 2000 >> gpurun_out/prof_plain.log 2>&1
timeout 300 python scripts/profile_integrator.py --steps 500 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lattice -c 1 -o gpurun_out/integ_wave python scripts/profile_integrator.py --steps 500 > gpurun_out/ncu_full.log 2>&1
echo all done
