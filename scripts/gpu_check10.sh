cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/profile_integrator.py --steps 2000 > gpurun_out/prof_plain.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python scripts/profile_integrator.py --steps 500 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lattice -c 1 -o gpurun_out/integ_v11 python scripts/profile_integrator.py --steps 500 > gpurun_out/ncu_full.log 2>&1
echo all done
