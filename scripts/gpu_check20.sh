cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python scripts/large_configs.py --config4 > gpurun_out/config4.jsonl 2> gpurun_out/config4.err
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_torchrun1.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v12.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
echo all done
