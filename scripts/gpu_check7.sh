cd $GRAFT_REPO_ROOT
timeout 1200 python scripts/scale_check.py --gens 2 > gpurun_out/scale.log 2>&1; echo "rc=$?" >> gpurun_out/scale.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v7.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo all done
