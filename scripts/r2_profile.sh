# Round-2 profiling pass (one GPU): cluster topology probe, variant timings of
# the 10^3 cluster integrator, the bench's ncu launch list, and ncu --set full
# captures of the bench-shape cluster kernel and the GA / decode kernels.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-r2p}
timeout -s KILL 120 scripts/cluster_probe > gpurun_out/${T}_cluster_probe.txt 2>&1
timeout -s KILL 120 scripts/microbench_dmma > gpurun_out/${T}_dmma.txt 2>&1
cp paper_2405_00698_b200/_lib/libvoxevo_b200.so /tmp/main.so
for rep in 1 2; do
for v in main $(ls _variants 2>/dev/null); do
  if [ $v = main ]; then cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; else cp _variants/$v/libvoxevo_b200.so paper_2405_00698_b200/_lib/libvoxevo_b200.so; fi
  echo -n "$v: " >> gpurun_out/${T}_variants.txt; timeout -s KILL 120 python scripts/profile_integrator.py --grid 10 --P 528 --steps 2000 2>&1 | tail -1 >> gpurun_out/${T}_variants.txt
done
done
cp /tmp/main.so paper_2405_00698_b200/_lib/libvoxevo_b200.so
if [ -z "${NO_NCU:-}" ]; then
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launch.log 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:cluster_vertex_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/${T}_cluster10_bench -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${T}_ncu_cluster.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:'decode_kernel|breed|mutate|hist_sel|diversity|stats_kernel|sample_kernel' --launch-count 12 -o gpurun_out/${T}_ga_decode -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${T}_ncu_ga.log 2>&1
fi
cat gpurun_out/${T}_cluster_probe.txt | head -30; cat gpurun_out/${T}_variants.txt; tail -3 gpurun_out/${T}_ncu_cluster.log gpurun_out/${T}_ncu_ga.log; ls -la gpurun_out/
