"""Short, ncu-friendly run of the config-2 integrator.

Builds the config-2 population's mass-spring systems on device (decode ->
component -> build) and runs the fused integrator for --steps steps (default
500, one launch), so `ncu --set full -k regex:integrate` replays a short
kernel.  Prints the updates/s of the launch (CUDA events).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00698_b200 as vx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--P", type=int, default=256)
    ap.add_argument("--grid", type=int, default=6)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    ctx = vx.Context(0)
    cfg = vx.EvolutionConfig(population=args.P, grid=(args.grid,) * 3, seed=42)
    st = vx.init_evolution(cfg, ctx)
    pop = st.population()
    g = args.grid
    mats, wts = vx.decode(pop["params"], pop["bmat"], cfg.arch, g, g, g, ctx)
    bodies = vx.largest_component(mats, g, g, g, ctx)
    batch = vx.build_mass_spring(bodies, wts, g, g, g, ctx=ctx)
    sim = vx.SimConfig(duration=args.steps * 1e-5)
    ctx.timing(True)
    for _ in range(args.reps):
        summ = batch.simulate(sim)
    ms, n = ctx.integrator_time()
    upd = sum(int(s.spring_updates) for s in summ)
    print(f"P={args.P} grid={g} steps={args.steps}: {upd} updates, {ms / n:.3f} ms/launch, "
          f"{upd / (ms / n * 1e-3):.4e} updates/s")


if __name__ == "__main__":
    main()
