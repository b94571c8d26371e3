"""BASELINE.json configs 3 and 4 on one B200 (device only, JSON lines).

  --config3: P=4096, 10^3, 50 generations (evolve_generation called 50 times,
             i.e. generations = 49 in the reference's run_loop convention),
             elite 0.3 / cx 0.4 / mutation 0.1, 0.1 / tournament 3, 5000
             steps; reports generations/s and spring updates/s.
  --config4: P=65536, 10^3, sharded over W GPUs: one GPU's share of a
             generation (vx_evo_begin(rank 0, W): decode + evaluate of every
             W-th child) timed for W in --worlds; the all-reduce of the
             exchange buffer and finish() are not part of the shard
             time (finish is timed separately on the full-population state).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00698_b200 as vx  # noqa: E402


def config3(gens, steps):
    ctx = vx.Context(0)
    cfg = vx.EvolutionConfig(population=4096, generations=gens - 1, grid=(10, 10, 10), seed=42,
                             sim=vx.SimConfig(duration=steps * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    total_upd, t_all = 0, 0.0
    for g in range(gens):
        t0 = time.perf_counter()
        rep = st.evolve_generation()
        dt = time.perf_counter() - t0
        total_upd += int(rep.spring_updates)
        t_all += dt
        print(json.dumps(dict(config="3", generation=rep.generation, seconds=dt, evaluations=rep.evaluations,
                              spring_updates=int(rep.spring_updates), best=rep.best, mean=rep.mean,
                              diversity=rep.diversity, integrator=ctx.last_integrator)), flush=True)
    print(json.dumps(dict(config="3 summary", population=4096, grid=10, steps=steps, generations=gens,
                          seconds=t_all, generations_per_s=gens / t_all, spring_updates=total_upd,
                          updates_per_s=total_upd / t_all)), flush=True)


def config4(worlds, steps):
    import torch
    ctx = vx.Context(0)
    P = 65536
    cfg = vx.EvolutionConfig(population=P, grid=(10, 10, 10), seed=42, sim=vx.SimConfig(duration=steps * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    xbuf = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device="cuda")  # [fitness|updates|packed grids]
    st.set_exchange_buffer(xbuf.data_ptr())
    for w in worlds:
        xbuf.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.begin(0, w)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        upd = int(xbuf[P:2 * P].sum().item())
        print(json.dumps(dict(config="4 shard", population=P, world=w, rank=0, seconds=dt, spring_updates=upd,
                              updates_per_s=upd / dt, integrator=ctx.last_integrator)), flush=True)
        t1 = time.perf_counter()
        st.finish()  # one GPU: the buffer holds rank 0's share only (timing of the replicated tail)
        ctx.synchronize()
        print(json.dumps(dict(config="4 finish", population=P, world=w, seconds=time.perf_counter() - t1,
                              note="merge + sort/stats/diversity/breed of the full population")), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config3", action="store_true")
    ap.add_argument("--config4", action="store_true")
    ap.add_argument("--gens", type=int, default=50)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--worlds", type=int, nargs="+", default=[8, 4, 2])
    a = ap.parse_args()
    if a.config3:
        config3(a.gens, a.steps)
    if a.config4:
        config4(a.worlds, a.steps)


if __name__ == "__main__":
    main()
