cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout -s KILL 300 python scripts/profile_integrator.py --steps 5000 > gpurun_out/prof23.log 2>&1
timeout -s KILL 300 python scripts/profile_integrator.py --steps 2000 --grid 10 --P 528 >> gpurun_out/prof23.log 2>&1
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench23.log 2>&1
echo all done
