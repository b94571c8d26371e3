cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "large or nondefault" > gpurun_out/pytest_stream.log 2>&1; rc=$?
echo "rc=$rc" >> gpurun_out/pytest_stream.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout -s KILL 300 python scripts/profile_integrator.py --steps 100 --grid 20 --P 148 > gpurun_out/prof21.log 2>&1
VX_INTEGRATOR=stream timeout -s KILL 300 python scripts/profile_integrator.py --steps 500 --grid 10 --P 296 >> gpurun_out/prof21.log 2>&1
echo all done
