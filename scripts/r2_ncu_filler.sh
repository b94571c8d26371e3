# ncu of the config-3 bench integrator with the device-launched filler: the
# launch list (cluster grid + its child), then --set full of the persistent
# cluster grid at the bench shape (generation 1)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${T}_ncu_launch.log
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:'cluster_vertex_|stream_sym_filler' --launch-skip 1 --launch-count 2 -o gpurun_out/${T}_cluster10_filler -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${T}_ncu_cluster.log 2>&1
echo "full rc=$?" >> gpurun_out/${T}_ncu_cluster.log
tail -5 gpurun_out/${T}_ncu_launch.log gpurun_out/${T}_ncu_cluster.log
