"""Population sharding through the LIBRARY across process boundaries.

Two processes, each with its own CUDA context on the one GPU, run the same
EvolutionState with vx_evo_set_exchange(rank, 2, fn): the library decodes and
evaluates only the rank's shard of the children and calls fn between begin
and finish; fn sums the exchange buffer over the ranks with gloo (host
copies).  Reports, populations and RNG streams must equal the
single-process run bit for bit — the reference's thread-count invariance
(test_evolution.cpp:196-215) across ranks.  The kernels of
the two ranks never wait on each other: the exchange is a host collective
between two complete device phases.

The NCCL path (vx_comm_create + vx_evo_set_comm, the product's own
communicator) runs here as a world-1 communicator — the all-reduce over one
rank is the identity, so the run must equal the unsharded one — and as a
real two-rank run only where two GPUs exist.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["VX_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2405_00698_b200 as vx
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
P, grid, steps, gens, mode = (int(os.environ["VX_P"]), int(os.environ["VX_GRID"]), int(os.environ["VX_STEPS"]),
                              int(os.environ["VX_GENS"]), os.environ["VX_MODE"])
dist.init_process_group("gloo")
dev = int(os.environ.get("VX_DEVICE_OF_RANK", "0")) * rank
ctx = vx.Context(dev)
cfg = vx.EvolutionConfig(population=P, generations=gens, grid=(grid,) * 3, seed=31,
                         sim=vx.SimConfig(duration=steps * 1e-5))
st = vx.init_evolution(cfg, ctx)
if mode == "gloo":
    torch.cuda.set_device(dev)
    xbuf = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device=f"cuda:{dev}")
    st.set_exchange_buffer(xbuf.data_ptr())
    def exchange(d_ptr, n):
        assert d_ptr == xbuf.data_ptr() and n == xbuf.numel()
        h = xbuf.cpu()
        dist.all_reduce(h)  # SUM over ranks, gloo on host copies
        xbuf.copy_(h)
        torch.cuda.synchronize()
    st.set_exchange(rank, world, exchange)
else:  # the library's own NCCL communicator
    obj = [vx.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = vx.Communicator(ctx, world, rank, obj[0])
    st.set_comm(comm)
reps = []
for g in range(gens):
    r = st.evolve_generation()
    reps.append([r.generation, r.best, r.mean, r.stddev, r.diversity, r.evaluations, float(r.spring_updates)])
pop = st.population()
np.savez(os.path.join(os.environ["VX_OUT"], f"rank{rank}.npz"), reps=np.array(reps), params=pop["params"],
         bmat=pop["bmat"], fitness=pop["fitness"], evaluated=pop["evaluated"],
         rng=np.frombuffer(st.rng_state().encode(), np.uint8))
if mode != "gloo":
    st.set_comm(None)
    comm.close()
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(tmp_path, world, mode, P, grid, steps, gens, device_of_rank=0):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = _free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, VX_ROOT=ROOT, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), VX_P=str(P), VX_GRID=str(grid), VX_STEPS=str(steps), VX_GENS=str(gens),
                   VX_MODE=mode, VX_OUT=str(tmp_path), VX_DEVICE_OF_RANK=str(device_of_rank))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    for p in procs:
        out, _ = p.communicate(timeout=900)
        assert p.returncode == 0, out[-3000:]
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]


def _single(vx, ctx, P, grid, steps, gens):
    cfg = vx.EvolutionConfig(population=P, generations=gens, grid=(grid,) * 3, seed=31,
                             sim=vx.SimConfig(duration=steps * 1e-5))
    st = vx.init_evolution(cfg, ctx)
    reps = []
    for _ in range(gens):
        r = st.evolve_generation()
        reps.append([r.generation, r.best, r.mean, r.stddev, r.diversity, r.evaluations, float(r.spring_updates)])
    pop = st.population()
    return dict(reps=np.array(reps), params=pop["params"], bmat=pop["bmat"], fitness=pop["fitness"],
                evaluated=pop["evaluated"], rng=np.frombuffer(st.rng_state().encode(), np.uint8))


def _assert_identical(got, want):
    for k in ("reps", "params", "bmat", "fitness", "evaluated", "rng"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)


@pytest.mark.parametrize("P,grid,steps,gens", [(256, 6, 300, 3), (512, 10, 100, 2)])
def test_two_processes_gloo_exchange_bit_identical(vx, ctx, tmp_path, P, grid, steps, gens):
    want = _single(vx, ctx, P, grid, steps, gens)
    ranks = _run_ranks(tmp_path, 2, "gloo", P, grid, steps, gens)
    for got in ranks:
        _assert_identical(got, want)


def test_nccl_world1_communicator_is_identity(vx, ctx, tmp_path):
    if not vx.Communicator.available():
        pytest.fail("NCCL (libnccl.so.2) not loadable on the GPU box")
    want = _single(vx, ctx, 128, 6, 300, 3)
    (got,) = _run_ranks(tmp_path, 1, "nccl", 128, 6, 300, 3)
    _assert_identical(got, want)


def test_nccl_two_gpus_bit_identical(vx, ctx, tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU: NCCL needs a distinct device per rank")
    want = _single(vx, ctx, 256, 6, 300, 3)
    ranks = _run_ranks(tmp_path, 2, "nccl", 256, 6, 300, 3, device_of_rank=1)
    for got in ranks:
        _assert_identical(got, want)
