# Round-2 GPU pass: the GPU suite (all failures listed), smoke, the C++
# drop-in demo, the default bench line and the reference arm.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout -s KILL 300 tests/cpp/_build/shim_demo > gpurun_out/${T}_shim.log 2>&1; echo "shim rc=$?" >> gpurun_out/${T}_shim.log
if [ -z "${NO_BENCH:-}" ]; then
s=$(date +%s); timeout -s KILL 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/${T}_bench.err
s=$(date +%s); timeout -s KILL 1200 python bench.py --impl reference ${BENCH_ARGS:-} > gpurun_out/${T}_bench_ref.log 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/${T}_bench_ref.err
fi
tail -3 gpurun_out/${T}_pytest_gpu.log; tail -2 gpurun_out/${T}_smoke.log; grep -c PASS gpurun_out/${T}_shim.log; grep FAIL gpurun_out/${T}_shim.log; tail -1 gpurun_out/${T}_shim.log
tail -2 gpurun_out/${T}_bench.err 2>/dev/null; tail -2 gpurun_out/${T}_bench_ref.err 2>/dev/null
