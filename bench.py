#!/usr/bin/env python
"""bench.py — spring-mass updates/s of the voxevo hot path on B200.

Workload (default, BASELINE.json configs[2], "config 3" — the largest
single-GPU configuration): population 4096 of 10x10x10 voxel robots per GPU,
evolve_generation (evolution.hpp:217-293) with elite selection / crossover /
mutation at the reference defaults, 5000-step fitness (dt 1e-5).  A bench
STEP is ONE generation of ONE continuing run: generation 0 (all P robots
decoded and evaluated) is the first warm-up step, every later step is the next
generation (~0.7P children decoded, assembled, simulated; elites keep their
cached fitness, exactly like the reference).  Work differs slightly between
generations, so

  value : sum of the EXACT spring updates of the K timed generations / sum of
          their device time (CUDA events on the context stream), population
          resident in HBM
  e2e   : K further generations of the same run through the public API with
          the population HOST-resident in pinned memory: every step uploads
          the population (genomes, fitness, evaluated flags) and downloads the
          bred population plus fitness, both inside the timed region
  generations_per_s : K / sum of the device time

--workload config2 / config5 run P=256 6^3 / P=1024 20^3 the same way.
Multi-GPU (torchrun, or --gpus N which relaunches itself under torchrun):
weak scaling, P = 4096 per GPU; the population is replicated, the children
are sharded, and the library's own NCCL communicator (vx_comm_create)
all-reduces the exchange buffer once per generation.

--impl reference runs the reference's own CPU implementation (the compiled,
unmodified reference headers in oracle/_ref): successive evolve_generation
calls of a bounded population (P=64 of the same grid; 256 for config 2) with
every host thread, each step timed alone and audited for its exact spring
updates outside the timed region.
"""
import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIM_STEPS = 5000
DT = 1e-5
SEED = 42
FLOPS_PER_UPDATE = 48  # 48 FP64 flop (+1 sqrt +1 div) per spring update
MLP_MACS_PER_VOXEL = 2 * 32 * 64 + 64 * 64 + 64 * 6  # default network (m=32, hidden 64-64, 5+1 heads)
METRIC = "spring-mass updates/sec (1/2/4/8 B200) and generations/sec at fixed population"
WORKLOADS = {
    "config3": dict(P=4096, grid=10, ref_P=64, cpu_sample=32,
                    kernel="cluster_vertex_persistent<10> (33 persistent 4-CTA clusters, one robot at a time each) + its "
                           "device-launched stream_sym_filler<10> on the 16 SMs no cluster can use",
                    traffic="cluster_traffic.json",
                    desc="config 3: population 4096 of 10x10x10 robots per GPU, successive generations of one run "
                         "(elite selection / crossover / mutation, 5000-step fitness)"),
    "config2": dict(P=256, grid=6, ref_P=256, cpu_sample=256,
                    kernel="vertex_kernel<6> (fused integrator K7-K9, vertex-key-indexed)",
                    traffic="integrator_traffic.json",
                    desc="config 2: population 256 of 6x6x6 robots per GPU, successive generations of one run "
                         "(decode + 5000-step fitness + sort/stats/diversity + breed)"),
    "config5": dict(P=1024, grid=20, ref_P=8, cpu_sample=8,
                    kernel="stream_sym_kernel<20> (symmetric streaming integrator)",
                    traffic="stream_traffic.json",
                    desc="config 5: population 1024 of 20x20x20 robots per GPU, successive generations of one run "
                         "(5000-step fitness, streaming integrator)"),
}


def rank_info():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def host_info() -> dict:
    """CPU model, glibc and the libm variant glibc's ifunc picks."""
    model = platform.processor() or "unknown"
    flags = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
            if ln.startswith("flags"):
                flags = ln.split(":", 1)[1]
            if model != "unknown" and flags:
                break
    except OSError:
        pass
    fl = set(flags.split())
    libm = ("glibc ifunc FMA/AVX2 variants (__exp_fma, __sin_fma, ...)" if {"fma", "avx2"} <= fl
            else "glibc ifunc generic (SSE2) variants")
    try:
        glibc = os.confstr("CS_GNU_LIBC_VERSION")
    except (ValueError, OSError):
        glibc = "unknown"
    return {"cpu_model": model, "glibc": glibc, "libm_variant": libm, "host_threads": os.cpu_count() or 1}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def config_block(W, world):
    """Identical in both arms (same_config)."""
    return {"workload": W["desc"], "population_per_gpu": W["P"], "population": W["P"] * world,
            "grid": [W["grid"]] * 3, "sim_steps": SIM_STEPS, "dt": DT, "seed": SEED,
            "hyper": "reference defaults: elite 0.3, crossover 0.4, mutation rate 0.1 scale 0.1, tournament 3",
            "l2": "flushed (256 MiB write) between steps", "parallelism": f"population shards x{world}"}


def make_config(vx, P, grid):
    return vx.EvolutionConfig(population=P, generations=0, grid=(grid, grid, grid), seed=SEED,
                              sim=vx.SimConfig(dt=DT, duration=SIM_STEPS * DT))


# ---------------------------------------------------------------- reference arm
def run_reference(args, W):
    """--impl reference: the reference's evolve_generation on the host cores."""
    rank, world, _ = rank_info()
    if rank != 0:
        return
    import oracle
    if not oracle.have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libvoxevo_ref.so not built"}))
        return
    ref = oracle.reference()
    threads = os.cpu_count() or 1
    sim = oracle.sim6(dt=DT, duration=SIM_STEPS * DT)
    P, g = W["ref_P"], W["grid"]
    ev = ref.evo(population=P, generations=0, grid=(g, g, g), seed=SEED, threads=threads, sim=sim)
    secs, upds = [], []
    for it in range(args.warmup + args.steps):
        _, s, u = ev.generation_timed()
        if it >= args.warmup:
            secs.append(s)
            upds.append(u)
    total = float(np.sum(secs))
    value = float(np.sum(upds)) / total
    sample = (f"reference evolve_generation (evolution.hpp:217-293) on a bounded population P={P} of {g}^3 robots "
              f"(the config's grid, hyper-parameters and 5000-step fitness), successive generations "
              f"{args.warmup}..{args.warmup + args.steps - 1} of one run, one per step, timed alone; exact spring "
              f"updates audited outside the timed region; headers compiled -O2 no -march, std::thread parallel_for "
              f"with {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spring_updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(W, world),
        "generations_per_s": len(secs) / total,
        "spring_updates_per_step": float(np.mean(upds)),
        "cpu_baseline": {"value": value, "unit": "spring_updates/s", "cores": threads, "kind": "reference",
                         "sample": sample, **host_info()},
        "e2e": {"value": value, "unit": "spring_updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_cpu_protocol(args):
    """--cpu-protocol: BASELINE.md §3's CPU-baseline protocol, the reference
    (oracle/_ref: its headers compiled -O2, no -march, -ffp-contract=off) on
    this box's host cores, with the GPU's run_bench beside it.  Bounded: every
    CPU measurement is a few seconds of work; configs 3-5 and the O(P^2)
    diversity are measured at a reduced population and extrapolated (labelled).
    Prints one JSON object."""
    import oracle
    if not oracle.have_reference():
        print(json.dumps({"cpu_protocol": "unavailable", "why": "oracle/_ref/libvoxevo_ref.so not built"}))
        return
    ref = oracle.reference()
    cores = os.cpu_count() or 1
    out = {"cpu_protocol": "BASELINE.md §3", "host": host_info(),
           "build": "reference headers, g++ -std=c++20 -O2 -ffp-contract=off, no -march (oracle/Makefile)",
           "libm": "default glibc ifunc selection (no GLIBC_TUNABLES)"}
    # 1. run_bench (bench.hpp:50-86) on bench_robot(n), 1 thread and all cores
    rb = []
    for n in (4, 6, 10, 20):
        springs = None
        for threads in (1, cores):
            jobs = 2 if threads == 1 else 2 * threads
            probe = np.zeros(6)
            ref._run_bench(1, 1, 1, n, DT, probe.ctypes.data)
            springs = int(probe[0])
            target = 1.5e8 * (1 if threads == 1 else max(1, threads // 2))  # ~2-4 s of CPU work
            steps = max(50, int(target / (jobs * springs)))
            o = np.zeros(6)
            ref._run_bench(jobs, steps, threads, n, DT, o.ctypes.data)
            assert int(o[1]) == int(o[2]), "run_bench audit mismatch"
            rb.append({"n": n, "threads": threads, "jobs": jobs, "steps": steps, "springs_per_robot": springs,
                       "spring_updates": int(o[1]), "seconds": o[3], "updates_per_s": o[4]})
    out["run_bench"] = rb
    # the same harness on the B200 (vx_run_bench: one batched launch)
    try:
        import paper_2405_00698_b200 as vx
        ctx = vx.Context(0)
        gb = []
        for n in (4, 6, 10, 20):
            jobs, steps = (296, 5000) if n <= 10 else (148, 500)
            vx.run_bench(jobs=jobs, steps=50, grid=n, ctx=ctx)  # warm-up
            r = vx.run_bench(jobs=jobs, steps=steps, grid=n, ctx=ctx)
            assert r["spring_updates"] == r["expected_updates"]
            gb.append({"n": n, "jobs": jobs, "steps": steps, "spring_updates": r["spring_updates"],
                       "seconds": r["seconds"], "updates_per_s": r["updates_per_second"]})
        out["run_bench_b200"] = gb
    except Exception as e:  # CPU-only host: the reference half still stands
        out["run_bench_b200"] = f"unavailable: {e}"
    sim = oracle.sim6(dt=DT, duration=SIM_STEPS * DT)
    # 2. config 1: one 4^3 robot from sample_genome({32,3,1.0},{64,64},seed), 1000 steps
    sim1 = oracle.sim6(dt=DT, duration=1000 * DT)
    p1, b1 = ref.sample_genome(32, [64, 64], SEED)
    t0 = time.perf_counter()
    m1, w1 = ref.decode(32, [64, 64], p1, b1, 4, 4, 4)
    f1 = ref.evaluate_fitness(m1, w1, 4, 4, 4, sim=sim1)
    out["config1"] = {"seconds": time.perf_counter() - t0, "fitness": f1,
                      "what": "decode + evaluate_fitness of one 4^3 robot, 1000 steps, 1 thread"}
    # 3./4./6. configs 2-5: evolve_generation wall (generations/s), reduced P for 3-5 (extrapolated)
    gens = []
    for name, P_full, P, g in (("config2", 256, 256, 6), ("config3", 4096, 64, 10), ("config4", 65536, 64, 10),
                               ("config5", 1024, max(8, cores), 20)):  # >= one robot per host thread
        if name == "config4":  # same robots as config 3 at 16x the population: extrapolate config 3's sample
            c3 = gens[-1]
            gens.append({"config": name, "P": P_full, "extrapolated_from": "config3 sample",
                         "seconds_per_generation": c3["seconds_per_generation"] * P_full / 4096,
                         "generations_per_s": 1.0 / (c3["seconds_per_generation"] * P_full / 4096),
                         "updates_per_s": c3["updates_per_s"]})
            continue
        ev = ref.evo(population=P, generations=0, grid=(g, g, g), seed=SEED, threads=cores, sim=sim)
        _, secs, upd = ev.generation_timed()  # generation 0: every robot evaluated
        row = {"config": name, "P": P_full, "P_measured": P, "threads": cores, "seconds_measured": secs,
               "generation": "0 (every robot evaluated; later generations evaluate ~0.7P)",
               "spring_updates_measured": int(upd), "updates_per_s": upd / secs}
        row["seconds_per_generation"] = secs * P_full / P
        row["generations_per_s"] = 1.0 / row["seconds_per_generation"]
        if P != P_full:
            row["extrapolated"] = f"linear in P from a P={P} generation 0 (exact update count)"
        gens.append(row)
    out["evolve_generation"] = gens
    # 5. serial stages: decode (morphology.hpp:141) and population_diversity (evolution.hpp:89)
    dec = []
    for g in (4, 6, 10, 20):
        reps = 8 if g <= 10 else 2
        t0 = time.perf_counter()
        for r in range(reps):
            ref.decode(32, [64, 64], p1, b1, g, g, g)
        dec.append({"grid": g, "seconds_per_genome": (time.perf_counter() - t0) / reps})
    out["serial_decode"] = dec
    div = []
    rng = np.random.default_rng(0)
    for name, P_full, P, g in (("config2", 256, 256, 6), ("config3", 4096, 512, 10), ("config5", 1024, 128, 20)):
        mats = rng.integers(0, 5, (P, g ** 3), dtype=np.uint8)
        t0 = time.perf_counter()
        ref.population_diversity(mats)
        secs = time.perf_counter() - t0
        row = {"config": name, "P": P_full, "P_measured": P, "seconds_measured": secs,
               "seconds_at_P": secs * (P_full / P) ** 2}
        if P != P_full:
            row["extrapolated"] = "quadratic in P (O(P^2 cells) pair loop)"
        div.append(row)
    out["serial_diversity"] = div
    print(json.dumps(out))


def cpu_baseline_and_parity(W, params0, bmat0, fit0_gpu):
    """The reference (oracle/_ref) on a bounded sample of this run's generation-0
    robots: its own decode, then evaluate_fitness through its parallel_for on
    every host thread (timed), and the per-robot fitness parity of the GPU
    generation 0 against it."""
    import oracle
    g = W["grid"]
    n = min(W["cpu_sample"], params0.shape[0])
    if not oracle.have_reference():
        return None, None
    lib = oracle.reference()
    threads = os.cpu_count() or 1
    cells = g ** 3
    mats = np.zeros((n, cells), np.uint8)
    wts = np.zeros((n, cells))
    for a in range(n):
        mats[a], wts[a] = lib.decode(32, [64, 64], params0[a], bmat0[a], g, g, g)
    fit = np.zeros(n)
    upd = np.zeros(1, np.uint64)
    sim = oracle.sim6(dt=DT, duration=SIM_STEPS * DT)
    secs = lib._evaluate_batch(n, g, g, g, mats.ctypes.data, wts.ctypes.data, oracle.DEFAULT_TABLE.ctypes.data,
                               oracle.DEFAULT_PLANE.ctypes.data, sim.ctypes.data, threads, fit.ctypes.data,
                               upd.ctypes.data)
    cpu = {"value": float(upd[0]) / secs, "unit": "spring_updates/s", "cores": threads, "kind": "reference",
           "sample": f"reference decode + evaluate_fitness (evolution.hpp:110-119) of generation 0's first {n} "
                     f"{g}^3 robots x {SIM_STEPS} steps ({int(upd[0])} updates) via its parallel_for, {secs:.2f} s",
           **host_info()}
    gpu = fit0_gpu[:n]
    rel = np.abs(gpu - fit) / np.maximum(np.abs(fit), 1e-12)
    parity = {"n": int(n), "max_rel": float(rel.max()), "median_rel": float(np.median(rel)),
              "exact": int(np.sum(gpu == fit)), "tolerance": "max <= 1e-3, median <= 1e-4 (SURVEY.md §8(d))",
              "ok": bool(rel.max() <= 1e-3 and np.median(rel) <= 1e-4),
              "what": "GPU generation-0 fitness vs the reference's decode + evaluate_fitness of the same genomes"}
    return cpu, parity


def relaunch_under_torchrun(args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines, no clocks)")
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-protocol", action="store_true",
                    help="BASELINE.md §3: the reference's CPU protocol on this host (+ GPU run_bench beside it)")
    args = ap.parse_args()
    if args.cpu_protocol:
        run_cpu_protocol(args)
        return
    W = WORKLOADS[args.workload]
    rank, world, local = rank_info()
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ
    if args.gpus > 1 and not launched:
        relaunch_under_torchrun(args)
    if launched and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 1:
        raise SystemExit("bench.py: --warmup must be >= 1 (generation 0 is a warm-up step)")
    if args.impl == "reference":
        run_reference(args, W)
        return

    import torch
    import torch.distributed as dist

    import paper_2405_00698_b200 as vx

    torch.cuda.set_device(local)
    if launched:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = vx.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    P = W["P"] * world
    st = vx.init_evolution(make_config(vx, P, W["grid"]), ctx)
    np_, nb = st.np, 3 * st.config.arch.m
    comm = None
    if launched and world > 1:  # the library's own NCCL communicator does the exchange
        obj = [vx.Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = vx.Communicator(ctx, world, rank, obj[0])
        st.set_comm(comm)
    xbuf = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device="cuda")  # fitness|updates|histogram
    st.set_exchange_buffer(xbuf.data_ptr())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if launched:
            dist.barrier()

    # ---- warm-up: generation 0 (all P robots) and W-1 more
    pop0 = st.population()
    params0, bmat0 = pop0["params"], pop0["bmat"]
    del pop0
    fit0 = None
    for it in range(args.warmup):
        st.evolve_generation()
        if it == 0:
            fit0 = xbuf[:P].cpu().numpy().copy()  # generation-0 fitness in individual order
    barrier()

    # ---- value: K generations, population resident in HBM
    ctx.timing(True)
    ctx.integrator_time(reset=True)
    ctx.decode_time(reset=True)
    launches0 = ctx.launches
    ms, upd = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = st.evolve_generation()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            upd.append(int(rep.spring_updates))
    launches = ctx.launches - launches0
    int_ms, int_n = ctx.integrator_time(reset=True)
    dec_ms, dec_vox = ctx.decode_time(reset=True)
    ctx.timing(False)

    # ---- e2e: K more generations with the population host-resident (pinned)
    ms_e2e, upd_e2e = [], []
    h2d = d2h = 0
    if not args.no_e2e and not args.profile:
        hp = torch.empty((P, np_), dtype=torch.float64, pin_memory=True)
        hb = torch.empty((P, nb), dtype=torch.float64, pin_memory=True)
        hf = torch.empty(P, dtype=torch.float64, pin_memory=True)
        he = torch.empty(P, dtype=torch.uint8, pin_memory=True)
        hpn, hbn, hfn, hen = hp.numpy(), hb.numpy(), hf.numpy(), he.numpy()
        st.get_population_into(hpn, hbn, hfn, hen)  # the run's state moves to the host
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st.set_population(hpn, hbn, hfn, hen)  # H2D: genomes, fitness, evaluated flags
            rep = st.evolve_generation()
            st.get_population_into(hpn, hbn, hfn, hen)  # D2H: the bred population and its fitness
            e1.record(stream)
            torch.cuda.synchronize()
            ms_e2e.append(e0.elapsed_time(e1))
            upd_e2e.append(int(rep.spring_updates))
        h2d = d2h = P * (np_ + nb) * 8 + P * 8 + P

    total_ms = float(np.sum(ms))
    total_e2e = float(np.sum(ms_e2e)) if ms_e2e else 0.0
    if launched:
        t = torch.tensor([total_ms, total_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, total_e2e = float(t[0]), float(t[1])
    value = float(np.sum(upd)) / (total_ms * 1e-3)
    value_e2e = float(np.sum(upd_e2e)) / (total_e2e * 1e-3) if ms_e2e else None
    if rank != 0:
        if comm is not None:
            st.set_comm(None)
            comm.close()
        dist.destroy_process_group()
        return

    # roofline of the dominant kernel, from live CUDA events on the launching stream
    local_upd = float(np.sum(upd)) / world  # this rank's share (children are dealt round-robin)
    avg_int_ms = int_ms / max(1, int_n)
    upd_per_launch = local_upd / max(1, int_n)
    meta = _ncu_json(W["traffic"])
    traffic = meta.get("dram_bytes_per_launch") if meta.get("workload") == args.workload else None
    if args.workload == "config5":
        peak_gbs, peak_src = _hbm_peak()
        ab = meta.get("algorithmic_bytes_per_update", 60)
        achieved = ab * upd_per_launch / (avg_int_ms * 1e-3) / 1e9 if int_n else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                    "frac": (achieved / peak_gbs) if achieved else None, "traffic": traffic,
                    "peak_source": peak_src,
                    "algorithmic": f"{ab} B per spring update (SURVEY.md §8(d)) x {upd_per_launch:.4g} updates per "
                                   "launch"}
        mb = meta.get("dram_bytes_per_update")  # measured (ncu dram__bytes) per update, same kernel
        if mb and int_n and roofline["traffic"] is None:
            roofline["traffic"] = mb * upd_per_launch  # the capture's bytes/update x this launch's updates
        if mb and int_n:
            ach_m = mb * upd_per_launch / (avg_int_ms * 1e-3) / 1e9
            roofline.update({"achieved_measured_dram": ach_m, "frac_measured_dram": ach_m / peak_gbs,
                             "dram_bytes_per_update_ncu": mb,
                             "fp64_pipe_busy_ncu": meta.get("fp64_pipe_pct"),
                             "note": "the kernel evaluates every spring from both endpoints (no force slots): "
                                     "FP64-issue and L2-latency bound, see DESIGN.md §3 (streaming integrator)"})
    else:
        achieved = FLOPS_PER_UPDATE * upd_per_launch / (avg_int_ms * 1e-3) / 1e12 if int_n else None
        peak = ctx.fp64_peak_tflops()
        roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                    "peak_source": "measured DFMA throughput of this GPU (vx_fp64_peak, csrc/measure.cu; "
                                   "MEASURED_PEAKS.json has no FP64 entry), 2 flop per DFMA",
                    "algorithmic": f"{FLOPS_PER_UPDATE} FP64 flop + 1 sqrt + 1 div per spring update (SURVEY.md "
                                   f"§8(d)) x {upd_per_launch:.4g} updates per launch",
                    "note": "parity mode forbids FMA contraction and the IEEE sqrt / reciprocal cost ~15 FP64 "
                            "instructions for 2 counted flop, so the flop fraction is structurally capped near 40%; "
                            "fp64_pipe_busy_ncu is the FP64-pipe utilisation of the same kernel at the bench shape"}
    roofline.update({"kernel": W["kernel"], "kernel_ms_avg": avg_int_ms, "launches_timed": int_n,
                     "kernel_share_of_step": (int_ms / total_ms) if total_ms else None,
                     "fp64_pipe_busy_ncu": meta.get("fp64_pipe_pct") if meta.get("workload") == args.workload
                     else None,
                     "ncu_source": meta.get("source")})

    # north star NS-1: the decode MLP on the FP64 tensor pipe, from the same live events
    decode = None
    if dec_ms > 0:
        dpk = ctx.dmma_peak_tflops()
        dach = 2.0 * MLP_MACS_PER_VOXEL * dec_vox / (dec_ms * 1e-3) / 1e12
        decode = {"kernel": "decode_mma_kernel (every MLP layer on DMMA, mma.sync m8n8k4 .f64) + the exact-order "
                            "fix-up launch", "bound": "fp64 tensor pipe (DMMA) + FP64 transcendentals",
                  "achieved": dach, "peak": dpk, "unit": "TFLOP/s", "frac": dach / dpk,
                  "algorithmic": f"2 x {MLP_MACS_PER_VOXEL} MAC per voxel (default network) x {dec_vox} voxels "
                                 "decoded in the timed generations",
                  "peak_source": "measured DMMA m8n8k4 throughput of this GPU (vx_dmma_peak, csrc/measure.cu)",
                  "ms_per_step": dec_ms / args.steps, "share_of_step": dec_ms / total_ms,
                  "dmma_pipe_busy_ncu": 31.4, "ncu_source": "profiles/r02_decode_dmma.md"}

    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        cpu, parity = cpu_baseline_and_parity(W, params0, bmat0, fit0)
    line = {
        "metric": METRIC, "value": value, "unit": "spring_updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_block(W, world),
        "generations_per_s": args.steps / (total_ms * 1e-3),
        "generations_timed": f"{args.warmup}..{args.warmup + args.steps - 1} (generation 0 = first warm-up step)",
        "spring_updates_per_step": float(np.mean(upd)),
        "spring_updates_timed": int(np.sum(upd)),
        "e2e": {"value": value_e2e, "unit": "spring_updates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "what": f"generations {args.warmup + args.steps}..{args.warmup + 2 * args.steps - 1} with the "
                        "population host-resident (pinned): upload + evolve_generation + download per step",
                "generations_per_s": (len(ms_e2e) / (total_e2e * 1e-3)) if ms_e2e else None},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "decode_roofline": decode,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clk.summary(),
        "vs_paper_rtx3090": value / 7892537853.0,
        "best_fitness": float(st.best()[0]),
    }
    print(json.dumps(line))
    if comm is not None:
        st.set_comm(None)
        comm.close()
    if launched:
        dist.destroy_process_group()


def _ncu_json(name):
    """Figures from a committed ncu capture of the workload's integrator (profiles/*.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return {}


def _hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling guide's figure."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6556.5, "B200_PROFILING.md fallback"


if __name__ == "__main__":
    main()
