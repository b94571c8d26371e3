"""Where a config-3 generation's wall time goes (development aid).

Runs generations of the bench workload through begin()/finish() and prints,
per generation: host time inside begin (queueing decode + evaluate), the
device time until the queued work drains, host time inside finish (sort,
stats, diversity, plan join, breeding) and the integrator's own event time.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=4096)
    ap.add_argument("--grid", type=int, default=10)
    ap.add_argument("--gens", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5000)
    args = ap.parse_args()
    import torch
    import paper_2405_00698_b200 as vx
    ctx = vx.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    g = args.grid
    cfg = vx.EvolutionConfig(population=args.P, generations=0, grid=(g, g, g), seed=42,
                             sim=vx.SimConfig(dt=1e-5, duration=args.steps * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    ctx.timing(True)
    for gen in range(args.gens):
        ctx.integrator_time(reset=True)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        t0 = time.perf_counter()
        e0.record(stream)
        st.begin(0, 1)
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rep = st.finish()
        t3 = time.perf_counter()
        e2.record(stream)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        ims, n = ctx.integrator_time(reset=True)
        print(f"gen {gen}: evals {rep.evaluations:5d}  begin host {1e3 * (t1 - t0):8.2f} ms  "
              f"drain {1e3 * (t2 - t1):8.2f} ms  finish host {1e3 * (t3 - t2):8.2f} ms  tail {1e3 * (t4 - t3):6.2f} ms | "
              f"gpu begin->drain {e0.elapsed_time(e1) + e1.elapsed_time(e2) - 0:8.2f} ms  integrator {ims:8.2f} ms "
              f"({n} launches)  total wall {1e3 * (t4 - t0):8.2f} ms")


if __name__ == "__main__":
    main()
