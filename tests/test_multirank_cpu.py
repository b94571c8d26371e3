"""Multi-rank protocol on CPU (gloo, world_size 2).

The GPU path shards a generation's children across ranks (vx_evo_begin): a
rank decodes and evaluates only the individuals it owns, then all-reduces
(SUM) the (2P + 5 cells)-double exchange buffer [fitness P | work counts P |
material histogram cells x 5] — zeros for what other ranks own — and breeds
identically everywhere (vx_evo_finish).  Here the same protocol runs with
the oracle as the per-rank evaluator: the reduced fitness must equal a
single-process evaluation bit for bit, the reduced histogram must give the
reference's population_diversity over all grids (evolution.hpp:89-105), and
the replicated breeding must give identical populations and RNG states on
every rank — the GPU analogue of the reference's thread-count invariance
(test_evolution.cpp:196-215).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

P, GRID = 8, 3
CELLS = GRID ** 3
SIM = None


def diversity_from_histogram(hist, P):
    """diversity_kernel (csrc/ga.cu): exact integer pair counts per cell."""
    h = np.asarray(hist, np.int64).reshape(-1, 5)
    pairs = P * (P - 1) // 2
    same = (h * (h - (h > 0)) // 2).sum()
    if P < 2 or len(h) == 0:
        return 0.0
    return (float(pairs * len(h) - same) / len(h)) / pairs


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2405_00698_b200 as vx

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = oracle.restatement()
    sim = oracle.sim6(dt=1e-4, duration=0.02)
    ev = lib.evo(population=P, generations=2, grid=(GRID,) * 3, hidden=(12, 12), m=8, seed=5, sim=sim)
    for gen in range(3):
        pop = ev.population()
        todo = [a for a in range(P) if not pop["evaluated"][a]]
        # decode is replicated; evaluation is sharded
        mats, wts = [], []
        for a in range(P):
            m, w = lib.decode(8, [12, 12], pop["params"][a], pop["bmat"][a], GRID, GRID, GRID)
            mats.append(m)
            wts.append(w)
        xbuf = torch.zeros(2 * P + 5 * CELLS, dtype=torch.float64)
        for a in vx.shard_indices(todo, rank, world):
            xbuf[a] = lib.evaluate_fitness(mats[a], wts[a], GRID, GRID, GRID, sim=sim)
            xbuf[P + a] = 1.0
        for a in vx.shard_indices(list(range(P)), rank, world):  # the grids this rank holds
            for c in range(CELLS):
                xbuf[2 * P + 5 * c + int(mats[a][c])] += 1.0
        dist.all_reduce(xbuf)
        fit = pop["fitness"].copy()
        for a in todo:
            fit[a] = xbuf[a].item()
        assert xbuf[P:2 * P].sum().item() == len(todo)  # every child evaluated exactly once
        assert xbuf[2 * P:].sum().item() == P * CELLS     # every grid counted exactly once
        div = diversity_from_histogram(xbuf[2 * P:].numpy().astype(np.int64), P)
        np.testing.assert_allclose(div, lib.population_diversity(np.stack(mats)), rtol=1e-13)
        ev.set_population(pop["params"], pop["bmat"], fit, np.ones(P, np.uint8), np.stack(mats), np.stack(wts))
        rep = ev.generation()
        np.save(os.path.join(out_dir, f"r{rank}_g{gen}_fit.npy"), fit)
        np.save(os.path.join(out_dir, f"r{rank}_g{gen}_params.npy"), ev.population()["params"])
        with open(os.path.join(out_dir, f"r{rank}_g{gen}_rng.txt"), "w") as f:
            f.write(ev.rng_state())
        with open(os.path.join(out_dir, f"r{rank}_g{gen}_rep.txt"), "w") as f:
            f.write(repr((rep["best"], rep["mean"], rep["diversity"])))
    dist.destroy_process_group()


def test_shard_indices_partition(vx):
    todo = list(range(3, 40, 3))
    for world in (1, 2, 3, 4, 8):
        parts = [vx.shard_indices(todo, r, world) for r in range(world)]
        flat = sorted(x for p in parts for x in p)
        assert flat == sorted(todo)
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_two_rank_generation_matches_single_process(tmp_path):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    # single-process reference run of the same generations
    import oracle
    lib = oracle.restatement()
    sim = oracle.sim6(dt=1e-4, duration=0.02)
    ev = lib.evo(population=P, generations=2, grid=(GRID,) * 3, hidden=(12, 12), m=8, seed=5, sim=sim)
    for gen in range(3):
        ev.generation()
        for r in (0, 1):
            np.testing.assert_array_equal(np.load(tmp_path / f"r{r}_g{gen}_params.npy"), ev.population()["params"])
            assert (tmp_path / f"r{r}_g{gen}_rng.txt").read_text() == ev.rng_state()
        np.testing.assert_array_equal(np.load(tmp_path / f"r0_g{gen}_fit.npy"), np.load(tmp_path / f"r1_g{gen}_fit.npy"))
        assert (tmp_path / f"r0_g{gen}_rep.txt").read_text() == (tmp_path / f"r1_g{gen}_rep.txt").read_text()
