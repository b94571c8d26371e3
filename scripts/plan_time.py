import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2405_00698_b200 as vx
ctx = vx.Context(0)
for world in [int(w) for w in os.environ.get("WORLDS", "1,2,4,8").split(",")]:
    P = 256 * world
    cfg = vx.EvolutionConfig(population=P, grid=(6, 6, 6), seed=42, sim=vx.SimConfig(duration=5000 * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    xb = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device="cuda")
    st.set_exchange_buffer(xb.data_ptr())
    for g in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.begin(0, world)
        ctx.synchronize()
        t1 = time.perf_counter()
        rep = st.finish()
        t2 = time.perf_counter()
        print(f"world {world} P {P} gen {g}: begin {1e3*(t1-t0):.1f} ms, finish {1e3*(t2-t1):.1f} ms, evals {rep.evaluations}", flush=True)
