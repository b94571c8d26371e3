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


def main(argv=None) -> int:
    """``python -m paper_2405_00698_b200 run.json [--resume checkpoint.json]``:
    the reference CLI's run / resume over this build (voxevo_main.cpp)."""
    import argparse
    from .serialize import load_run_config
    ap = argparse.ArgumentParser(prog="python -m paper_2405_00698_b200")
    ap.add_argument("config")
    ap.add_argument("--resume", default=None)
    a = ap.parse_args(argv)
    rc = load_run_config(a.config)
    if a.resume:
        resume_run(a.resume, rc, log=sys.stdout)
    else:
        start_run(rc, log=sys.stdout)
    return 0


if __name__ == "__main__":
    sys.exit(main())
