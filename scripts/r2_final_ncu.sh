# final round-2 evidence: config-2 and config-5 bench lines, then ncu --set full
# of the config-3 integrator (persistent clusters + device-launched filler) at
# the bench shape
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
T=${TAG:-r2z}
timeout -s KILL 900 python bench.py --workload config5 --steps 3 --warmup 3 > gpurun_out/${T}_bench5.log 2> gpurun_out/${T}_bench5.err; echo "rc=$?" >> gpurun_out/${T}_bench5.err
timeout -s KILL 600 python bench.py --workload config2 > gpurun_out/${T}_bench2.log 2> gpurun_out/${T}_bench2.err; echo "rc=$?" >> gpurun_out/${T}_bench2.err
timeout -s KILL 1700 ncu --set full --clock-control none --import-source on -k regex:'cluster_vertex_' --launch-skip 1 --launch-count 1 -o gpurun_out/${T}_cluster10 -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${T}_ncu.log
tail -c 600 gpurun_out/${T}_bench5.log; tail -c 400 gpurun_out/${T}_bench2.log; tail -2 gpurun_out/${T}_ncu.log
