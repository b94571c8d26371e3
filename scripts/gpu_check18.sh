cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_api.py -q -x > gpurun_out/pytest_cluster.log 2>&1; rc=$?
echo "rc=$rc" >> gpurun_out/pytest_cluster.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout -s KILL 300 python scripts/profile_integrator.py --steps 500 --grid 10 --P 296 > gpurun_out/prof_cluster.log 2>&1
timeout -s KILL 300 python scripts/profile_integrator.py --steps 2000 --grid 10 --P 528 >> gpurun_out/prof_cluster.log 2>&1
timeout -s KILL 600 python scripts/large_configs.py --config4 > gpurun_out/config4.jsonl 2> gpurun_out/config4.err
echo all done
