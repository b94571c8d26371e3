# One GPU pass a maintainer (or the round driver) can run on a B200 box:
# the GPU parity suite, the smoke test, the integrator timings of every
# kernel (6^3 lattice, 10^3 cluster, 20^3 streaming) and the bench line.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 300 python scripts/profile_integrator.py --steps 5000 > gpurun_out/integrators.log 2>&1
timeout -s KILL 300 python scripts/profile_integrator.py --steps 2000 --grid 10 --P 528 >> gpurun_out/integrators.log 2>&1
timeout -s KILL 300 python scripts/profile_integrator.py --steps 100 --grid 20 --P 148 >> gpurun_out/integrators.log 2>&1
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/integrators.log; tail -1 gpurun_out/bench.log | cut -c1-300
