"""Multi-rank protocol on CPU (gloo, world_size 2).

The GPU path shards a generation's children across ranks (vx_evo_begin): a
rank decodes and evaluates only the individuals it owns, then all-reduces
(SUM) the (2P + P W)-double exchange buffer [fitness P | work counts P |
packed grids P x W, 12 four-bit cells per double] — zeros for what other
ranks own — and breeds identically everywhere (vx_evo_finish).  Here the
same protocol runs with the oracle as the per-rank evaluator: the reduced
fitness must equal a single-process evaluation bit for bit, the reduced
packed grids must give back every decoded grid exactly (so every rank
computes the reference's population_diversity, evolution.hpp:89-105, on the
same grids in the same sorted order), and
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


W = (CELLS + 11) // 12  # diversity_words (csrc/diversity.cu)


def pack_grid(mat):
    """pack_kernel (csrc/diversity.cu): 12 four-bit cells per double (< 2^48, exact)."""
    out = np.zeros(W)
    for w in range(W):
        v = 0
        for k in range(12):
            c = 12 * w + k
            if c < len(mat):
                v |= (int(mat[c]) & 0xF) << (4 * k)
        out[w] = float(v)
    return out


def unpack_grid(words):
    return np.array([(int(words[c // 12]) >> (4 * (c % 12))) & 0xF for c in range(CELLS)], np.uint8)


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
        xbuf = torch.zeros(2 * P + P * W, dtype=torch.float64)
        for a in vx.shard_indices(todo, rank, world):
            xbuf[a] = lib.evaluate_fitness(mats[a], wts[a], GRID, GRID, GRID, sim=sim)
            xbuf[P + a] = 1.0
        for a in vx.shard_indices(list(range(P)), rank, world):  # the grids this rank holds
            xbuf[2 * P + a * W:2 * P + (a + 1) * W] = torch.from_numpy(pack_grid(mats[a]))
        dist.all_reduce(xbuf)
        fit = pop["fitness"].copy()
        for a in todo:
            fit[a] = xbuf[a].item()
        assert xbuf[P:2 * P].sum().item() == len(todo)  # every child evaluated exactly once
        packed = xbuf[2 * P:].numpy().reshape(P, W)
        for a in range(P):  # every grid gathered exactly once, bit for bit
            np.testing.assert_array_equal(unpack_grid(packed[a]), mats[a])
        order = np.argsort(-fit, kind="stable")  # the sorted population the diversity is taken over
        div = lib.population_diversity(np.stack([unpack_grid(packed[a]) for a in order]))
        assert div == lib.population_diversity(np.stack([mats[a] for a in order]))
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
