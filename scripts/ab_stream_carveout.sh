cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do for co in none 0 25 30 40 60 100; do
 echo -n "carveout=$co: "; if [ $co = none ]; then timeout 120 python scripts/profile_integrator.py --grid 20 --P 148 --steps 200 2>&1 | tail -1; else VX_STREAM_CARVEOUT=$co timeout 120 python scripts/profile_integrator.py --grid 20 --P 148 --steps 200 2>&1 | tail -1; fi
done; done
