cd ${GRAFT_REPO_ROOT:-.}
timeout -s KILL 600 env VX_STREAM_TMA=1 python -m pytest tests/test_gpu_configs.py -q -x -k "20" 2>&1 | tail -1
for rep in 1 2 3; do for m in 1 0; do echo -n "tma=$m: "; VX_STREAM_TMA=$m timeout -s KILL 120 python scripts/profile_integrator.py --grid 20 --P 148 --steps 200 2>&1 | tail -1; done; done
