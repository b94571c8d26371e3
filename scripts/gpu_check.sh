set -x
cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | head -20 >> gpurun_out/smi.txt; ldd --version | head -1 >> gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
