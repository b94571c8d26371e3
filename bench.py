#!/usr/bin/env python
"""bench.py — spring-mass updates/s of the voxevo hot path on B200.

(--workload config3 / config5 run BASELINE configs 3 / 5 under the same
contract: one generation of P=4096 10^3 / P=1024 20^3 robots per step.)

Workload (BASELINE.json configs[1], "config 2"): population 256 of 6x6x6 voxel
robots per GPU, ONE generation = decode (Fourier encoding + MLP) -> largest
component -> mass-spring assembly -> 5000-step fused integrator (dt 1e-5) ->
fitness -> stable sort / stats / diversity -> elite + tournament / crossover /
mutation breeding.  A bench "step" is one such generation from the same
synthetic generation-0 population (genomes sampled on device from seed 42 with
the reference's mt19937_64 streams), so every step does identical work.

  value : whole-job spring updates/s with the genomes already resident in HBM
  e2e   : the same through the public API with the genomes copied host(pinned)
          -> device and the fitness vector copied back inside the timed region
Multi-GPU (torchrun): weak scaling, 256 robots evaluated per GPU; the
population (256*N) is replicated, children are sharded, one NCCL all-reduce
of the fitness exchange buffer per generation.

--impl reference runs the reference's own CPU implementation (the compiled,
unmodified reference headers in oracle/_ref) through evolve_generation with
all host threads on the same config.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_PER_GPU = 256
GRID = 6
SIM_STEPS = 5000
# --workload: the default is config 2 (BASELINE.json configs[1], the driver's
# line); configs 3 and 5 run one generation of their population per step
WORKLOADS = {
    "config2": dict(P=256, grid=6, kernel="vertex_kernel<6> (fused integrator K7-K9, vertex-key-indexed)",
                    desc="config 2: P=256 6x6x6 per GPU, 1 generation (decode + 5000-step fitness + sort/stats/"
                         "diversity + breed)"),
    "config3": dict(P=4096, grid=10, kernel="cluster_vertex_kernel<10> (4-CTA thread-block cluster per robot)",
                    desc="config 3: P=4096 10x10x10 per GPU, 1 of the 50 generations per step (decode + "
                         "5000-step fitness + sort/stats/diversity + breed)"),
    "config5": dict(P=1024, grid=20, kernel="stream_sym_kernel<20> (symmetric streaming integrator)",
                    desc="config 5: P=1024 20x20x20 per GPU, 1 generation (decode + 5000-step fitness + sort/"
                         "stats/diversity + breed)"),
}
CPU_SAMPLE_MAX = 256  # robots in the bounded cpu_baseline sample
DT = 1e-5
SEED = 42
FLOPS_PER_UPDATE = 48  # 48 FP64 flop (+1 sqrt +1 div) per spring update
METRIC = "spring-mass updates/sec (1/2/4/8 B200) and generations/sec at fixed population"


def rank_info():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


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
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
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


def flush_l2(torch, buf):
    buf.zero_()  # 256 MiB > 126 MB L2


def make_config(vx, P):
    return vx.EvolutionConfig(population=P, generations=0, grid=(GRID, GRID, GRID), seed=SEED,
                              sim=vx.SimConfig(dt=DT, duration=SIM_STEPS * DT))


def cpu_baseline_sample(grids, weights):
    """Reference evaluate_fitness over the generation's 256 raw grids through
    its own parallel_for with all host threads (oracle/_ref)."""
    import oracle
    lib = oracle.reference() if oracle.have_reference() else None
    kind = "reference"
    threads = os.cpu_count() or 1
    n = grids.shape[0]
    fit = np.zeros(n)
    upd = np.zeros(1, np.uint64)
    sim = oracle.sim6(dt=DT, duration=SIM_STEPS * DT)
    if lib is None:  # restatement (single-threaded port)
        lib = oracle.restatement()
        kind, threads = "port", 1
        t0 = time.perf_counter()
        for a in range(n):
            fit[a] = lib.evaluate_fitness(grids[a], weights[a], GRID, GRID, GRID, sim=sim)
        secs = time.perf_counter() - t0
        return None, dict(kind=kind, cores=1, secs=secs)
    g = np.ascontiguousarray(grids, np.uint8)
    w = np.ascontiguousarray(weights, np.float64)
    secs = lib._evaluate_batch(n, GRID, GRID, GRID, g.ctypes.data, w.ctypes.data, oracle.DEFAULT_TABLE.ctypes.data,
                               oracle.DEFAULT_PLANE.ctypes.data, sim.ctypes.data, threads, fit.ctypes.data,
                               upd.ctypes.data)
    return int(upd[0]), dict(kind=kind, cores=threads, secs=secs, fitness=fit)


def run_reference(args):
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
    P = P_PER_GPU
    ev = ref.evo(population=P, generations=0, grid=(GRID, GRID, GRID), seed=SEED, threads=threads, sim=sim)
    pop0 = ev.population()
    # exact work audit of one generation (outside the timed region)
    mats = np.zeros((P, GRID ** 3), np.uint8)
    wts = np.zeros((P, GRID ** 3))
    for a in range(P):
        mats[a], wts[a] = ref.decode(32, [64, 64], pop0["params"][a], pop0["bmat"][a], GRID, GRID, GRID)
    upd, _ = cpu_baseline_sample(mats, wts)
    times = []
    for it in range(args.warmup + args.steps):
        ev.set_population(pop0["params"], pop0["bmat"])  # generation-0 state, nothing cached
        ev.set_rng_state(oracle.reference().rng_state(SEED, P))
        t0 = time.perf_counter()
        ev.generation()
        dt_s = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt_s)
    total = float(np.sum(times))
    value = upd * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spring_updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.desc, "population": P, "grid": [GRID] * 3, "sim_steps": SIM_STEPS, "dt": DT,
                   "seed": SEED},
        "generations_per_s": len(times) / total,
        "cpu_baseline": {"value": value, "unit": "spring_updates/s", "cores": threads, "kind": "reference",
                         "sample": f"full evolve_generation (P={P}, {GRID}^3, {SIM_STEPS} steps), reference "
                                   "headers compiled -O2 no -march, std::thread parallel_for"},
        "e2e": {"value": value, "unit": "spring_updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines, no clocks)")
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    global P_PER_GPU, GRID
    W = WORKLOADS[args.workload]
    P_PER_GPU, GRID = W["P"], W["grid"]
    args.kernel, args.desc = W["kernel"], W["desc"]
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2405_00698_b200 as vx

    rank, world, local = rank_info()
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # launched by torchrun (any N)
    torch.cuda.set_device(local)
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = vx.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    P = P_PER_GPU * world
    st = vx.init_evolution(make_config(vx, P), ctx)
    np_ = st.np
    nb = 3 * st.config.arch.m
    pop0 = st.population()  # generation-0 genomes sampled on device (K14)
    init_params = torch.from_numpy(pop0["params"]).cuda()
    init_bmat = torch.from_numpy(pop0["bmat"]).cuda()
    del pop0
    xbuf = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device="cuda")  # fitness|updates|histogram
    st.set_exchange_buffer(xbuf.data_ptr())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    host_params = torch.empty((P, np_), dtype=torch.float64, pin_memory=True)
    host_bmat = torch.empty((P, nb), dtype=torch.float64, pin_memory=True)
    host_params.copy_(init_params)
    host_bmat.copy_(init_bmat)
    host_fit = torch.empty(P, dtype=torch.float64, pin_memory=True)

    def generation(e2e: bool):
        if e2e:
            init_params.copy_(host_params, non_blocking=True)
            init_bmat.copy_(host_bmat, non_blocking=True)
        st.load_population_dev(init_params.data_ptr(), init_bmat.data_ptr())
        st.set_rng_state(_seed_state)
        st.begin(rank, world)
        if distributed:
            dist.all_reduce(xbuf)
        rep = st.finish()
        if e2e:
            host_fit.copy_(xbuf[:P], non_blocking=False)
        return rep

    # RNG stream position of init_evolution's output (breeding replays identically each step)
    _seed_state = st.rng_state()

    def timed(n, e2e):
        ms, reps = [], []
        for _ in range(n):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            if distributed:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            reps.append(generation(e2e))
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return ms, reps

    for _ in range(args.warmup):
        generation(False)
    torch.cuda.synchronize()
    ctx.timing(True)
    ctx.integrator_time(reset=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        ms, reps = timed(args.steps, e2e=False)
    launches = ctx.launches - launches0
    int_ms, int_n = ctx.integrator_time(reset=True)
    ctx.timing(False)
    ms_e2e, reps_e2e = timed(args.steps, e2e=True)

    total_ms = float(np.sum(ms))
    total_e2e = float(np.sum(ms_e2e))
    if distributed:
        t = torch.tensor([total_ms, total_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, total_e2e = float(t[0]), float(t[1])
    upd_per_step = int(reps[0].spring_updates)  # whole job (exchange buffer is all-reduced)
    assert all(int(r.spring_updates) == upd_per_step for r in reps + reps_e2e), "work differs between steps"
    value = upd_per_step * args.steps / (total_ms * 1e-3)
    value_e2e = upd_per_step * args.steps / (total_e2e * 1e-3)
    if rank != 0:
        dist.destroy_process_group()
        return

    # roofline of the dominant kernel (the fused integrator), from live CUDA events
    local_upd = upd_per_step // world
    avg_int_ms = int_ms / max(1, int_n)
    achieved_tf = FLOPS_PER_UPDATE * local_upd / (avg_int_ms * 1e-3) / 1e12 if int_n else None
    peak_tf = ctx.fp64_peak_tflops()
    # the dominant kernel's roofline: FP64-issue bound on chip (configs 2, 3),
    # HBM bound for the streaming integrator (config 5)
    prof = {"config2": "integrator_traffic.json", "config3": "cluster_traffic.json",
            "config5": "stream_traffic.json"}[args.workload]
    meta = _ncu_json(prof)
    launch_upd = local_upd
    traffic = None
    if meta.get("dram_bytes_per_launch") is not None and args.workload == "config2":
        traffic = meta["dram_bytes_per_launch"]  # captured at the config-2 launch shape (batch load dominated)
    elif meta.get("dram_bytes_per_update") is not None:
        traffic = meta["dram_bytes_per_update"] * launch_upd
    if args.workload == "config5":
        peak_gbs, peak_src = _hbm_peak()
        ab = meta.get("algorithmic_bytes_per_update", 60)
        achieved_gbs = ab * launch_upd / (avg_int_ms * 1e-3) / 1e9 if int_n else None
        roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak_gbs, "unit": "GB/s",
                    "frac": (achieved_gbs / peak_gbs) if achieved_gbs else None, "traffic": traffic,
                    "kernel": args.kernel, "kernel_ms_avg": avg_int_ms,
                    "kernel_share_of_step": (int_ms / total_ms) if total_ms else None, "peak_source": peak_src,
                    "algorithmic": f"{ab} B per spring update (SURVEY.md §8(d)) x {launch_upd} updates per launch",
                    "fp64_pipe_busy_ncu": meta.get("fp64_pipe_pct")}
    else:
        roofline = {"bound": "fp64", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": (achieved_tf / peak_tf) if achieved_tf else None, "traffic": traffic,
                    "kernel": args.kernel, "kernel_ms_avg": avg_int_ms,
                    "kernel_share_of_step": (int_ms / total_ms) if total_ms else None,
                    "peak_source": "measured DFMA throughput on this GPU (vx_fp64_peak; MEASURED_PEAKS.json has no "
                                   "FP64 entry), 2 flop/DFMA",
                    "algorithmic": f"{FLOPS_PER_UPDATE} FP64 flop + 1 sqrt + 1 div per spring update x "
                                   f"{local_upd} updates per launch",
                    "fp64_pipe_busy_ncu": meta.get("fp64_pipe_pct"),
                    "note": "parity mode forbids FMA contraction and IEEE sqrt/1/x cost ~15 FP64 instructions for 2 "
                            "counted flop, so the flop fraction is structurally capped near 40%; fp64_pipe_busy_ncu "
                            "is the FP64-pipe utilisation of the same kernel from the committed ncu capture"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        pop = st.population()  # after the last step: elites keep grids -> re-decode for the sample
        ns = min(P, CPU_SAMPLE_MAX if GRID <= 6 else 32)  # bounded: ~2-20 s of host work
        mats, wts = vx.decode(init_params[:ns].cpu().numpy(), init_bmat[:ns].cpu().numpy(), st.config.arch, GRID,
                              GRID, GRID, ctx)
        upd, meta = cpu_baseline_sample(mats, wts)
        cpu = {"value": (upd / meta["secs"]) if upd else None, "unit": "spring_updates/s", "cores": meta["cores"],
               "kind": meta["kind"],
               "sample": f"evaluate_fitness over {mats.shape[0]} of this config's decoded {GRID}^3 robots x "
                         f"{SIM_STEPS} steps ({upd} updates) via the reference's parallel_for, {meta['secs']:.2f} s"}
        del pop
    h2d = P * (np_ + nb) * 8
    d2h = P * 8 + P * 8 + 3 * 8 + 8 + 4
    line = {
        "metric": METRIC, "value": value, "unit": "spring_updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.desc, "population": P, "grid": [GRID] * 3,
                   "sim_steps": SIM_STEPS, "dt": DT, "seed": SEED, "l2": "flushed (256 MiB write) between steps",
                   "parallelism": f"population shards x{world}"},
        "generations_per_s": args.steps / (total_ms * 1e-3),
        "spring_updates_per_step": upd_per_step,
        "e2e": {"value": value_e2e, "unit": "spring_updates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "vs_paper_rtx3090": value / 7892537853.0,
        "best_fitness_gen0": reps[0].best,
    }
    print(json.dumps(line))
    if distributed:
        dist.destroy_process_group()


def _ncu_json(name):
    """Figures from a committed ncu capture of the workload's integrator (profiles/*.json)."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        return json.load(open(path))
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
