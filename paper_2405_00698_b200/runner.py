"""run_loop and its artifacts, and the rule-based advisor, for the
device-resident evolution state (host side; citations are to
/root/reference/proj/include/voxevo/):

* ``ScriptedAdvisor`` — advisor.hpp:25-55: diversity collapse boosts mutation
  rate and scale, stagnation boosts crossover, the proposal is clamped.
* ``run_loop`` / ``start_run`` / ``resume_run`` — runner.hpp:62-94: one
  evolve_generation per generation index 0..generations inclusive, a
  checkpoint every ``checkpoint_stride`` generations, then checkpoint.json,
  curves.csv, best_genome.json and the config echo config.json in
  ``out_dir`` (artifact_paths, runner.hpp:25-28).
* ``run_config_to_json`` — to_json(RunConfig) (config.hpp:106-147).

The LLM and replay advisors (advisor_http.hpp, advisor.hpp replay) are HTTP /
audit-log policy outside the hot path: a run config naming
them parses, but ``make_advisor`` refuses to run it.
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass
from typing import Optional, TextIO

from . import ADVISOR_WINDOW, Context, EvolutionState, GenerationReport, HyperParams, VoxevoError, init_evolution
from .serialize import (LLM_DEFAULTS, RunConfig, _struct_to_json, hyper_params_to_json, load_run, save_genome,
                        save_json_file, save_run, sim_config_to_json, write_curves_csv)


@dataclass
class RunArtifacts:
    """RunArtifacts / artifact_paths (runner.hpp:17-28)."""
    dir: str
    curves: str
    checkpoint: str
    best_genome: str
    config_echo: str


def artifact_paths(out_dir: str) -> RunArtifacts:
    return RunArtifacts(out_dir, out_dir + "/curves.csv", out_dir + "/checkpoint.json",
                        out_dir + "/best_genome.json", out_dir + "/config.json")


def advisor_consults_done(history_len: int) -> int:
    """advisor_consults_done (runner.hpp:33-36)."""
    return history_len - ADVISOR_WINDOW if history_len > ADVISOR_WINDOW else 0


class ScriptedAdvisor:
    """ScriptedAdvisor (advisor.hpp:25-55), an AdvisorFn."""

    def __init__(self, diversity_floor: float = 0.05, stagnation_eps: float = 1e-6, mutation_boost: float = 1.5,
                 crossover_boost: float = 1.25):
        self.diversity_floor = diversity_floor
        self.stagnation_eps = stagnation_eps
        self.mutation_boost = mutation_boost
        self.crossover_boost = crossover_boost

    def __call__(self, window: list, current: HyperParams) -> Optional[HyperParams]:
        if not window:
            return None
        nxt = current.copy()
        fired = False
        if window[-1].diversity < self.diversity_floor:
            nxt.mutation_rate *= self.mutation_boost
            nxt.mutation_scale *= self.mutation_boost
            fired = True
        if len(window) >= 2 and window[-1].best - window[0].best < self.stagnation_eps:
            nxt.crossover_rate *= self.crossover_boost
            fired = True
        if not fired:
            return None
        return nxt.clamp()


def make_advisor(rc: RunConfig, consults_done: int = 0):
    """make_advisor (runner.hpp:38-50)."""
    del consults_done  # only the LLM / replay advisors are stateful
    if rc.advisor == "scripted":
        return ScriptedAdvisor()
    if rc.advisor in ("llm", "replay"):
        raise VoxevoError(f"advisor '{rc.advisor}' is HTTP / audit-log policy outside this build (DESIGN.md §7)")
    return None


def run_config_to_json(rc: RunConfig) -> dict:
    """to_json(RunConfig) (config.hpp:106-147)."""
    e = rc.evolution
    j = {"population": int(e.population), "generations": int(e.generations),
         "grid": [int(e.grid_w), int(e.grid_h), int(e.grid_d)], "hidden_widths": list(e.arch.widths),
         "encoding": {"m": int(e.arch.m), "sigma": float(e.arch.sigma)}, "tournament_size": int(e.tournament_size),
         "threads": int(e.threads), "seed": int(e.seed), "params": hyper_params_to_json(e.initial_params),
         "materials": _struct_to_json(e.materials), "plane": _struct_to_json(e.plane),
         "sim": sim_config_to_json(e.sim), "advisor": rc.advisor, "replay_audit": rc.replay_audit,
         "out_dir": rc.out_dir, "checkpoint_stride": int(rc.checkpoint_stride)}
    llm = dict(LLM_DEFAULTS)
    llm.update({k: v for k, v in rc.llm.items() if k in LLM_DEFAULTS})
    j["llm"] = llm
    return j


def log_report(r: GenerationReport) -> str:
    """log_report (runner.hpp:52-60), one line."""
    p = r.params
    return ("gen %4d  best %.6f  mean %.6f  std %.6f  div %.3f  evals %3d  mr %.4g ms %.4g cx %.4g ef %.4g  [%.2fs]"
            % (r.generation, r.best, r.mean, r.stddev, r.diversity, r.evaluations, p.mutation_rate,
               p.mutation_scale, p.crossover_rate, p.elite_fraction, r.wall_time))


def run_loop(st: EvolutionState, rc: RunConfig, log: Optional[TextIO] = None) -> EvolutionState:
    """run_loop (runner.hpp:62-82): generations st.generation..config.generations."""
    os.makedirs(rc.out_dir, exist_ok=True)
    paths = artifact_paths(rc.out_dir)
    save_json_file(paths.config_echo, run_config_to_json(rc))
    advisor = make_advisor(rc, advisor_consults_done(len(st.history)))
    while st.generation <= st.config.generations:
        rep = st.evolve_generation(advisor)
        if log is not None:
            log.write(log_report(rep) + "\n")
        if rc.checkpoint_stride > 0 and rep.generation % rc.checkpoint_stride == 0:
            save_run(paths.checkpoint, st)
    save_run(paths.checkpoint, st)
    write_curves_csv(paths.curves, st.history)
    _, bp = st.best()
    if bp is not None:
        save_genome(paths.best_genome, bp, st._best_bmat(), st.config.arch)
    return st


def start_run(rc: RunConfig, ctx: Optional[Context] = None, log: Optional[TextIO] = None) -> EvolutionState:
    """start_run (runner.hpp:84-86)."""
    return run_loop(init_evolution(rc.evolution, ctx), rc, log)


def resume_run(checkpoint_path: str, rc: RunConfig, ctx: Optional[Context] = None,
               log: Optional[TextIO] = None) -> EvolutionState:
    """resume_run (runner.hpp:88-92)."""
    return run_loop(load_run(checkpoint_path, ctx), rc, log)


def _fmt_g(x: float) -> str:
    """std::ostream's default double format (precision 6, %g)."""
    return "%g" % x


def print_summary(st: EvolutionState, rc: RunConfig, out: TextIO = sys.stdout):
    """print_summary (voxevo_main.cpp:43-50)."""
    paths = artifact_paths(rc.out_dir)
    best_f, best_p = st.best()
    out.write("done: %d generations, best fitness %s m\n" % (len(st.history), _fmt_g(best_f)))
    out.write("  curves:     %s\n" % paths.curves)
    out.write("  checkpoint: %s\n" % paths.checkpoint)
    if best_p is not None:
        out.write("  champion:   %s\n" % paths.best_genome)


def _add_overrides(cmd, with_population=True):
    """CommonOverrides::add_to (voxevo_main.cpp:23-32)."""
    cmd.add_argument("--seed", type=int)
    cmd.add_argument("--generations", type=int)
    if with_population:
        cmd.add_argument("--population", type=int)
    cmd.add_argument("--threads", type=int)
    cmd.add_argument("--advisor", choices=["off", "scripted", "llm", "replay"])
    cmd.add_argument("--out", dest="out_dir")


def cmd_run(a) -> int:
    """cmd_run (voxevo_main.cpp:52-60): defaults, then the config file, then flags."""
    from .serialize import load_run_config
    rc = load_run_config(a.config) if a.config else RunConfig()
    e = rc.evolution
    if a.seed is not None:
        e.seed = a.seed
    if a.generations is not None:
        e.generations = a.generations
    if a.population is not None:
        e.population = a.population
    if a.threads is not None:
        e.threads = a.threads
    if a.advisor is not None:
        rc.advisor = a.advisor
    if a.out_dir is not None:
        rc.out_dir = a.out_dir
    st = start_run(rc, log=sys.stdout)
    print_summary(st, rc)
    return 0


def cmd_resume(a) -> int:
    """cmd_resume (voxevo_main.cpp:62-77): search settings stay with the
    checkpoint unless a flag overrides them."""
    from .serialize import load_run_config
    rc = load_run_config(a.config) if a.config else RunConfig()
    st = load_run(a.checkpoint)
    if a.generations is not None:
        st.config.generations = a.generations
    if a.threads is not None:
        st.config.threads = a.threads
    if a.advisor is not None:
        rc.advisor = a.advisor
    if a.out_dir is not None:
        rc.out_dir = a.out_dir
    st = run_loop(st, rc, sys.stdout)
    print_summary(st, rc)
    return 0


def cmd_bench(a) -> int:
    """cmd_bench (voxevo_main.cpp:79-101) over the device run_bench: the same
    line with the device in place of the worker-thread count."""
    from . import run_bench
    r = run_bench(a.jobs, a.steps, a.grid, a.dt)
    sys.stdout.write("device %2d: %d steps x %d jobs, %d springs/robot -> %d updates in %.3fs (%.3g/s)%s\n"
                     % (0, a.steps, a.jobs, r["springs_per_robot"], r["spring_updates"], r["seconds"],
                        r["updates_per_second"], "  [DIVERGED]" if r["diverged"] else ""))
    if r["spring_updates"] != r["expected_updates"]:
        sys.stderr.write("update count mismatch: expected %d\n" % r["expected_updates"])
        return 1
    if a.compare_single:
        sys.stderr.write("--compare-single: the device path has no worker-thread count; "
                         "bench.py --impl reference times the reference CPU build\n")
    return 0


def cmd_export(a) -> int:
    """cmd_export (voxevo_main.cpp:103-126): decode (and keep the largest
    component unless --full) on the device, then the reference's formats."""
    from . import decode, largest_component
    from .export import export_mesh_obj, export_voxel_listing
    from .serialize import load_genome
    params, bmat, arch = load_genome(a.genome)
    w, h, d = a.grid
    mats, wts = decode(params[None], bmat[None], arch, w, h, d)
    if not a.full:
        mats = largest_component(mats, w, h, d)
    occupied = int((mats[0] != 0).sum())
    if occupied == 0:
        sys.stderr.write("genome decodes to an empty robot at %dx%dx%d\n" % (w, h, d))
        return 1
    if a.out:
        export_mesh_obj(a.out, mats[0], w, h, d, a.edge)
        sys.stdout.write("mesh:   %s\n" % a.out)
    if a.voxels:
        export_voxel_listing(a.voxels, mats[0], wts[0], w, h, d)
        sys.stdout.write("voxels: %s\n" % a.voxels)
    sys.stdout.write("voxels occupied: %d\n" % occupied)
    return 0


def main(argv=None) -> int:
    """The reference CLI (voxevo_main.cpp:130-190) over this build:

      python -m paper_2405_00698_b200 run [--config c.json] [--seed --generations --population --threads
                                           --advisor --out]
      python -m paper_2405_00698_b200 resume --checkpoint ck.json [--config c.json] [--generations --threads
                                              --advisor --out]
      python -m paper_2405_00698_b200 bench [--jobs 16 --steps 2000 --grid 4 --dt 1e-5 --threads N
                                             --compare-single]
      python -m paper_2405_00698_b200 export-mesh --genome g.json [--out robot.obj --voxels v.txt
                                                   --grid W H D --full --edge 0.1]

    Errors print ``error: <what>`` and exit 1, like the reference's catch-all."""
    import argparse
    from . import MaterialTable, VoxevoError
    from .export import ExportError
    from .serialize import CheckpointError, ConfigError
    ap = argparse.ArgumentParser(prog="python -m paper_2405_00698_b200",
                                 description="voxevo: evolve simulated soft voxel robots")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="Start an evolution run")
    run.add_argument("--config")
    _add_overrides(run)
    res = sub.add_parser("resume", help="Continue from a checkpoint")
    res.add_argument("--checkpoint", required=True)
    res.add_argument("--config")
    _add_overrides(res, with_population=False)
    res.set_defaults(seed=None)
    ben = sub.add_parser("bench", help="Measure simulator throughput")
    ben.add_argument("--jobs", type=int, default=16)
    ben.add_argument("--steps", type=int, default=2000)
    ben.add_argument("--threads", type=int, default=1)
    ben.add_argument("--grid", type=int, default=4)
    ben.add_argument("--dt", type=float, default=1e-5)
    ben.add_argument("--compare-single", action="store_true")
    exp = sub.add_parser("export-mesh", help="Write a genome's morphology as OBJ")
    exp.add_argument("--genome", required=True)
    exp.add_argument("--out", default="robot.obj")
    exp.add_argument("--voxels", default="")
    exp.add_argument("--grid", type=int, nargs=3, default=[5, 5, 5])
    exp.add_argument("--full", action="store_true")
    exp.add_argument("--edge", type=float, default=MaterialTable().voxel_edge)
    a = ap.parse_args(argv)
    for name in ("jobs", "steps", "threads", "grid"):
        if a.cmd == "bench" and getattr(a, name) <= 0:
            ap.error("--%s must be positive" % name)
    for path in (getattr(a, "config", None), getattr(a, "checkpoint", None), getattr(a, "genome", None)):
        if path and not os.path.isfile(path):
            ap.error("file does not exist: %s" % path)
    try:
        return {"run": cmd_run, "resume": cmd_resume, "bench": cmd_bench, "export-mesh": cmd_export}[a.cmd](a)
    except (VoxevoError, CheckpointError, ConfigError, ExportError, ValueError, OSError) as e:
        sys.stderr.write("error: %s\n" % e)
        return 1


if __name__ == "__main__":
    sys.exit(main())
