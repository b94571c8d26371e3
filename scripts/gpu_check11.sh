cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/profile_integrator.py --steps 500 --grid 10 --P 296 > gpurun_out/prof_plain.log 2>&1
VX_INTEGRATOR=generic timeout 300 python scripts/profile_integrator.py --steps 500 --grid 10 --P 296 >> gpurun_out/prof_plain.log 2>&1
timeout 300 python scripts/profile_integrator.py --steps 100 --grid 20 --P 148 >> gpurun_out/prof_plain.log 2>&1
timeout 1200 python scripts/scale_check.py > gpurun_out/scale.log 2>&1
echo all done
