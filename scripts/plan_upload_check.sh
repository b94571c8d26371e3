# breeding / sharded-generation / advisor parity after moving the plan upload
# into the plan thread, then the finish() wait at P = 256 x world (6^3)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
T=${TAG:-pu}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_shard.py tests/test_gpu_advisor.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
VX_EVO_TRACE=1 timeout -s KILL 600 python scripts/plan_time.py > gpurun_out/${T}_plan.txt 2>&1
timeout -s KILL 600 python scripts/plan_time.py > gpurun_out/${T}_plan_notrace.txt 2>&1
tail -3 gpurun_out/${T}_tests.log; grep -v "mut copy" gpurun_out/${T}_plan.txt; cat gpurun_out/${T}_plan_notrace.txt
