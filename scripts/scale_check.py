"""One full generation at the large BASELINE.json configs (device only).

  config 3 shape: P=4096, 10x10x10, 5000 steps (one generation of the 50)
  config 5 shape: P=1024, 20x20x20, 5000 steps
Prints one JSON line per config with the generation time, exact spring
updates and updates/s.  --quick uses shorter horizons.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00698_b200 as vx  # noqa: E402


def run(P, grid, steps, gens=1):
    ctx = vx.Context(0)
    cfg = vx.EvolutionConfig(population=P, grid=(grid,) * 3, seed=42, sim=vx.SimConfig(duration=steps * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    ctx.timing(True)
    out = []
    for g in range(gens):
        t0 = time.perf_counter()
        rep = st.evolve_generation()
        dt = time.perf_counter() - t0
        ms, n = ctx.integrator_time()
        out.append(dict(config=f"P={P} {grid}^3 {steps} steps", generation=rep.generation, seconds=dt,
                        integrator_ms=ms, spring_updates=int(rep.spring_updates),
                        updates_per_s=rep.spring_updates / dt, evaluations=rep.evaluations, best=rep.best,
                        diversity=rep.diversity))
        print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--gens", type=int, default=1)
    a = ap.parse_args()
    steps = 500 if a.quick else 5000
    run(4096, 10, steps, a.gens)
    run(1024, 20, steps, a.gens)


if __name__ == "__main__":
    main()
