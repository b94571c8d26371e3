cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python scripts/large_configs.py --config4 > gpurun_out/config4.jsonl 2> gpurun_out/config4.err
timeout -s KILL 900 python scripts/large_configs.py --config3 > gpurun_out/config3.jsonl 2> gpurun_out/config3.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:lattice_kernel -c 1 -o gpurun_out/integ_v12 python scripts/profile_integrator.py --steps 500 > gpurun_out/ncu_v12.log 2>&1
echo all done
