"""Config files and checkpoints for the device-resident evolution state.

Host-side mirror of the reference's file formats (citations are to
/root/reference/proj/include/voxevo/):

* ``run_config_from_json`` — the lenient, defaulting run-config parser
  (config.hpp:31-127): every key optional, unknown keys ignored, ``grid`` must
  be ``[w, h, d]``, ``advisor`` one of off | scripted | llm | replay, else
  ``ConfigError`` (config_error, config.hpp:13-15).
* checkpoints — the strict component serializers (serialize.hpp:42-262) and
  the ``{magic, version, kind, checksum, payload}`` container whose checksum
  is the FNV-1a hash of the payload's canonical dump (serialize.hpp:264-292).
  ``dumps`` reproduces nlohmann::json's ``dump()`` byte for byte (sorted keys,
  no whitespace, its shortest round-trip number format), so a checkpoint the
  reference wrote loads here, one written here loads in the reference, and
  save/load/save is byte-stable (tests/test_serialize.py pins all three
  against the reference itself).
* ``curves_csv`` — the per-generation CSV (serialize.hpp:316-343).

Decoded grids are not stored (serialize.hpp:211-213); a resumed state decodes
every individual again on its next generation, exactly as the reference does.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from . import (NMAT, Arch, Context, EvolutionConfig, EvolutionState, GenerationReport, GroundPlane, HyperParams,
               MaterialTable, SimConfig, _lib, param_count)

CHECKPOINT_MAGIC = "voxevo"  # kCheckpointMagic (serialize.hpp:20)
CHECKPOINT_VERSION = 1       # kCheckpointVersion (serialize.hpp:21)
ADVISORS = ("off", "scripted", "llm", "replay")
# LlmAdvisorConfig defaults (advisor_http.hpp:22-34): parsed and echoed, never contacted
LLM_DEFAULTS = {"url": "http://127.0.0.1:8080", "path": "/v1/chat/completions", "model": "advisor-model",
                "api_key_env": "VOXEVO_LLM_KEY", "temperature": 0.0, "max_retries": 2, "backoff_base_ms": 1000,
                "connect_timeout_s": 5, "read_timeout_s": 30, "allow_material_multipliers": False,
                "audit_path": ""}
_LLM_KIND = {"temperature": float, "max_retries": int, "backoff_base_ms": int, "connect_timeout_s": int,
             "read_timeout_s": int, "allow_material_multipliers": bool}


class ConfigError(RuntimeError):
    """config_error (config.hpp:13-15)."""


class CheckpointError(RuntimeError):
    """checkpoint_error (serialize.hpp:16-18)."""


# ------------------------------------------------------ canonical JSON dump
def format_doubles_text(values, sep: str = ",") -> str:
    """nlohmann::json number text of each double, joined by `sep` (vx_format_doubles)."""
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        return ""
    cap = 26 * v.size + 1
    buf = C.create_string_buffer(cap)
    n = _lib().vx_format_doubles(v.ctypes.data, v.size, b",", buf, cap)
    if n < 0 or n >= cap:
        raise RuntimeError("vx_format_doubles failed")
    text = buf.raw[:n].decode()
    return text if sep == "," else text.replace(",", sep)


def format_doubles(values) -> list:
    """nlohmann::json number text of each double (vx_format_doubles)."""
    text = format_doubles_text(values)
    return text.split(",") if text else []


def _fmt_double(x: float) -> str:
    return format_doubles([x])[0]


def _is_float_list(seq) -> bool:
    return len(seq) > 0 and isinstance(seq[0], (float, np.floating)) and \
        all(isinstance(x, (float, np.floating)) and not isinstance(x, bool) for x in seq)


def _dump(v: Any, out: list, indent: Optional[int], level: int):
    if v is None:
        out.append("null")
    elif v is True:
        out.append("true")
    elif v is False:
        out.append("false")
    elif isinstance(v, (int, np.integer)):
        out.append(str(int(v)))
    elif isinstance(v, (float, np.floating)):
        out.append(_fmt_double(float(v)))
    elif isinstance(v, str):
        out.append(json.dumps(v, ensure_ascii=False))
    elif isinstance(v, dict):
        if not v:
            out.append("{}")
            return
        keys = sorted(v)
        if indent is None:
            out.append("{")
            for i, key in enumerate(keys):
                if i:
                    out.append(",")
                out.append(json.dumps(key, ensure_ascii=False) + ":")
                _dump(v[key], out, None, 0)
            out.append("}")
        else:
            pad, inner = " " * (indent * level), " " * (indent * (level + 1))
            out.append("{\n")
            for i, key in enumerate(keys):
                if i:
                    out.append(",\n")
                out.append(inner + json.dumps(key, ensure_ascii=False) + ": ")
                _dump(v[key], out, indent, level + 1)
            out.append("\n" + pad + "}")
    elif isinstance(v, (list, tuple, np.ndarray)):
        seq = v if isinstance(v, np.ndarray) else list(v)
        if len(seq) == 0:
            out.append("[]")
            return
        if (isinstance(seq, np.ndarray) and seq.dtype == np.float64) or _is_float_list(seq):
            # genome tensors: one library call per tensor, numbers never contain ','
            if indent is None:
                out.append("[" + format_doubles_text(seq) + "]")
            else:
                pad, inner = " " * (indent * level), " " * (indent * (level + 1))
                out.append("[\n" + inner + format_doubles_text(seq, ",\n" + inner) + "\n" + pad + "]")
            return
        if indent is None:
            out.append("[")
            for i, x in enumerate(seq):
                if i:
                    out.append(",")
                _dump(x, out, None, 0)
            out.append("]")
        else:
            pad, inner = " " * (indent * level), " " * (indent * (level + 1))
            out.append("[\n")
            for i, x in enumerate(seq):
                if i:
                    out.append(",\n")
                out.append(inner)
                _dump(x, out, indent, level + 1)
            out.append("\n" + pad + "]")
    else:
        raise TypeError(f"cannot serialise {type(v).__name__}")


def dumps(v: Any, indent: Optional[int] = None) -> str:
    """nlohmann::json::dump(indent) of a JSON value held as Python objects
    (ints stay integers, floats are doubles)."""
    out: list = []
    _dump(v, out, indent, 0)
    return "".join(out)


def fnv1a64_hex(data: str) -> str:
    """fnv1a64_hex (serialize.hpp:23-35) over the UTF-8 bytes."""
    b = data.encode()
    return "%016x" % _lib().vx_fnv1a64(b, len(b))


# --------------------------------------------------------------- configs
def _get(j: dict, key: str, default, kind=None):
    """nlohmann json::value(key, default): the stored value when present."""
    if key not in j:
        return default
    v = j[key]
    if kind is float:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise ConfigError(f"{key}: expected a number")
        return float(v)
    if kind is int:
        if isinstance(v, bool) or not isinstance(v, int):
            raise ConfigError(f"{key}: expected an integer")
        return int(v)
    if kind is bool:
        if not isinstance(v, bool):
            raise ConfigError(f"{key}: expected a boolean")
        return v
    if kind is str:
        if not isinstance(v, str):
            raise ConfigError(f"{key}: expected a string")
        return v
    return v


@dataclass
class RunConfig:
    """RunConfig (config.hpp:19-26).  ``llm`` holds the LlmAdvisorConfig fields
    (the HTTP advisor itself is out of scope)."""
    evolution: EvolutionConfig = field(default_factory=EvolutionConfig)
    advisor: str = "off"
    llm: dict = field(default_factory=lambda: dict(LLM_DEFAULTS))
    replay_audit: str = ""
    out_dir: str = "runs/latest"
    checkpoint_stride: int = 1


def run_config_from_json(j: Any) -> RunConfig:
    """run_config_from_json (config.hpp:31-127): lenient and defaulting."""
    if not isinstance(j, dict):
        raise ConfigError("run config must be a JSON object")
    rc = RunConfig()
    e = rc.evolution
    e.population = _get(j, "population", e.population, int)
    e.generations = _get(j, "generations", e.generations, int)
    if "grid" in j:
        g = j["grid"]
        if not isinstance(g, list) or len(g) != 3:
            raise ConfigError("grid must be [w, h, d]")
        e.grid_w, e.grid_h, e.grid_d = (int(x) for x in g)
    widths = e.arch.widths
    if "hidden_widths" in j:
        widths = [int(x) for x in j["hidden_widths"]]
    m, sigma = e.arch.m, e.arch.sigma
    if "encoding" in j:
        enc = j["encoding"]
        m = _get(enc, "m", m, int)
        sigma = _get(enc, "sigma", sigma, float)
    e.arch = Arch.make(m, widths, sigma)
    e.tournament_size = _get(j, "tournament_size", e.tournament_size, int)
    e.threads = _get(j, "threads", e.threads, int)
    e.seed = _get(j, "seed", e.seed, int)
    if "params" in j:
        p = j["params"]
        hp = e.initial_params
        for key in ("mutation_rate", "mutation_scale", "crossover_rate", "elite_fraction"):
            setattr(hp, key, _get(p, key, getattr(hp, key), float))
        if "material_multipliers" in p:
            mm = p["material_multipliers"]
            if not isinstance(mm, list) or len(mm) != 3:
                raise ConfigError("material_multipliers must have 3 entries")
            hp.material_multipliers = type(hp.material_multipliers)(*[float(x) for x in mm])
    for key, obj in (("materials", e.materials), ("plane", e.plane)):
        if key in j:
            for f, _ in obj._fields_:
                setattr(obj, f, _get(j[key], f, getattr(obj, f), float))
    if "sim" in j:
        s = j["sim"]
        for f in ("gravity", "dt", "duration", "actuation_frequency"):
            setattr(e.sim, f, _get(s, f, getattr(e.sim, f), float))
        for f in ("enable_gravity", "enable_contact"):
            setattr(e.sim, f, int(_get(s, f, bool(getattr(e.sim, f)), bool)))
    rc.advisor = _get(j, "advisor", rc.advisor, str)
    if rc.advisor not in ADVISORS:
        raise ConfigError("advisor must be off, scripted, llm, or replay")
    if "llm" in j:
        for key, default in LLM_DEFAULTS.items():
            rc.llm[key] = _get(j["llm"], key, default, _LLM_KIND.get(key, str))
    rc.replay_audit = _get(j, "replay_audit", rc.replay_audit, str)
    rc.out_dir = _get(j, "out_dir", rc.out_dir, str)
    rc.checkpoint_stride = _get(j, "checkpoint_stride", rc.checkpoint_stride, int)
    return rc


def load_run_config(path: str) -> RunConfig:
    """load_run_config (config.hpp:150-152): the file is read by
    load_json_file, so an unreadable file or bad JSON is a CheckpointError and
    a bad value a ConfigError, as in the reference."""
    return run_config_from_json(load_json_file(path))


# ---------------------------------------------------- component serializers
def _f(x) -> float:
    return float(x)


def hyper_params_to_json(p: HyperParams) -> dict:
    """to_json(HyperParams) (serialize.hpp:101-107)."""
    return {"mutation_rate": _f(p.mutation_rate), "mutation_scale": _f(p.mutation_scale),
            "crossover_rate": _f(p.crossover_rate), "elite_fraction": _f(p.elite_fraction),
            "material_multipliers": [_f(x) for x in p.material_multipliers]}


def _num(j: dict, key: str, err=CheckpointError) -> float:
    try:
        v = j[key]
    except (KeyError, TypeError) as exc:
        raise err(f"missing key: {key}") from exc
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise err(f"{key}: expected a number")
    return float(v)


def _int(j: dict, key: str) -> int:
    try:
        v = j[key]
    except (KeyError, TypeError) as exc:
        raise CheckpointError(f"missing key: {key}") from exc
    if isinstance(v, bool) or not isinstance(v, int):
        raise CheckpointError(f"{key}: expected an integer")
    return int(v)


def _bool(j: dict, key: str) -> bool:
    try:
        v = j[key]
    except (KeyError, TypeError) as exc:
        raise CheckpointError(f"missing key: {key}") from exc
    if not isinstance(v, bool):
        raise CheckpointError(f"{key}: expected a boolean")
    return v


def _at(j: dict, key: str):
    try:
        return j[key]
    except (KeyError, TypeError) as exc:
        raise CheckpointError(f"missing key: {key}") from exc


def hyper_params_from_json(j: dict) -> HyperParams:
    """hyper_params_from_json (serialize.hpp:109-117); not clamped, like the reference."""
    mm = _at(j, "material_multipliers")
    if not isinstance(mm, list) or len(mm) != 3:
        raise CheckpointError("material_multipliers must have 3 entries")
    p = HyperParams(mutation_rate=_num(j, "mutation_rate"), mutation_scale=_num(j, "mutation_scale"),
                    crossover_rate=_num(j, "crossover_rate"), elite_fraction=_num(j, "elite_fraction"))
    p.material_multipliers = type(p.material_multipliers)(*[float(x) for x in mm])
    return p


def report_to_json(r: GenerationReport) -> dict:
    """to_json(GenerationReport) (serialize.hpp:119-125)."""
    return {"generation": int(r.generation), "params": hyper_params_to_json(r.params), "best": _f(r.best),
            "mean": _f(r.mean), "stddev": _f(r.stddev), "diversity": _f(r.diversity),
            "evaluations": int(r.evaluations), "wall_time": _f(r.wall_time)}


def report_from_json(j: dict) -> GenerationReport:
    """report_from_json (serialize.hpp:127-138)."""
    r = GenerationReport()
    r.generation = _int(j, "generation")
    r.params = hyper_params_from_json(_at(j, "params"))
    for k in ("best", "mean", "stddev", "diversity", "wall_time"):
        setattr(r, k, _num(j, k))
    r.evaluations = _int(j, "evaluations")
    return r


def _struct_to_json(obj) -> dict:
    return {f: _f(getattr(obj, f)) for f, _ in obj._fields_}


def _struct_from_json(cls, j: dict):
    o = cls()
    for f, _ in cls._fields_:
        setattr(o, f, _num(j, f))
    return o


def sim_config_to_json(c: SimConfig) -> dict:
    """to_json(SimConfig) (serialize.hpp:140-147)."""
    return {"gravity": _f(c.gravity), "dt": _f(c.dt), "duration": _f(c.duration),
            "actuation_frequency": _f(c.actuation_frequency), "enable_gravity": bool(c.enable_gravity),
            "enable_contact": bool(c.enable_contact)}


def sim_config_from_json(j: dict) -> SimConfig:
    """sim_config_from_json (serialize.hpp:149-158)."""
    return SimConfig(gravity=_num(j, "gravity"), dt=_num(j, "dt"), duration=_num(j, "duration"),
                     actuation_frequency=_num(j, "actuation_frequency"),
                     enable_gravity=_bool(j, "enable_gravity"), enable_contact=_bool(j, "enable_contact"))


def evolution_config_to_json(c: EvolutionConfig) -> dict:
    """to_json(EvolutionConfig) (serialize.hpp:194-208)."""
    return {"population": int(c.population), "generations": int(c.generations),
            "grid": [int(c.grid_w), int(c.grid_h), int(c.grid_d)], "hidden_widths": list(c.arch.widths),
            "encoding": {"m": int(c.arch.m), "d": 3, "sigma": _f(c.arch.sigma)},
            "tournament_size": int(c.tournament_size), "threads": int(c.threads), "seed": int(c.seed),
            "initial_params": hyper_params_to_json(c.initial_params), "materials": _struct_to_json(c.materials),
            "plane": _struct_to_json(c.plane), "sim": sim_config_to_json(c.sim)}


def evolution_config_from_json(j: dict) -> EvolutionConfig:
    """evolution_config_from_json (serialize.hpp:210-228), strict."""
    c = EvolutionConfig()
    c.population = _int(j, "population")
    c.generations = _int(j, "generations")
    g = _at(j, "grid")
    if not isinstance(g, list) or len(g) != 3:
        raise CheckpointError("grid must be [w, h, d]")
    c.grid_w, c.grid_h, c.grid_d = (int(x) for x in g)
    enc = _at(j, "encoding")
    if _int(enc, "d") != 3:
        raise CheckpointError("only 3-D encodings are supported")
    c.arch = Arch.make(_int(enc, "m"), [int(x) for x in _at(j, "hidden_widths")], _num(enc, "sigma"))
    c.tournament_size = _int(j, "tournament_size")
    c.threads = _int(j, "threads")
    c.seed = _int(j, "seed")
    c.initial_params = hyper_params_from_json(_at(j, "initial_params"))
    c.materials = _struct_from_json(MaterialTable, _at(j, "materials"))
    c.plane = _struct_from_json(GroundPlane, _at(j, "plane"))
    c.sim = sim_config_from_json(_at(j, "sim"))
    return c


def _layer_shapes(arch: Arch) -> list:
    """(in, out) of every layer in param_tensors() order (genome.hpp:57-81)."""
    shapes, prev = [], 2 * arch.m
    for w in arch.widths:
        shapes.append((prev, w))
        prev = w
    shapes.append((prev, NMAT))  # head_material
    shapes.append((prev, 1))     # head_weight
    return shapes


def genome_to_json(params: np.ndarray, bmat: np.ndarray, arch: Arch) -> dict:
    """to_json(Genome) (serialize.hpp:78-86) from the flat device layout."""
    layers, o = [], 0
    for fan_in, fan_out in _layer_shapes(arch):
        w = params[o:o + fan_in * fan_out]
        o += fan_in * fan_out
        b = params[o:o + fan_out]
        o += fan_out
        layers.append({"in": fan_in, "out": fan_out, "w": np.asarray(w, np.float64).tolist(),
                       "b": np.asarray(b, np.float64).tolist()})
    return {"encoding": {"m": int(arch.m), "d": 3, "sigma": _f(arch.sigma)},
            "b_matrix": np.asarray(bmat, np.float64).tolist(),
            "hidden": layers[:-2], "head_material": layers[-2], "head_weight": layers[-1]}


def _layer_from_json(j: dict, shape) -> tuple:
    """layer_from_json (serialize.hpp:64-76): sizes must match the declared shape."""
    fan_in, fan_out = _int(j, "in"), _int(j, "out")
    w, b = _at(j, "w"), _at(j, "b")
    if len(w) != fan_in * fan_out or len(b) != fan_out:
        raise CheckpointError("layer tensor sizes do not match declared shape")
    if (fan_in, fan_out) != tuple(shape):
        raise CheckpointError("layer shape does not match the run's architecture")
    return w, b


def genome_from_json(j: dict, arch: Arch) -> tuple:
    """genome_from_json (serialize.hpp:88-99) -> (flat params, b_matrix)."""
    enc = _at(j, "encoding")
    if _int(enc, "m") != arch.m or _int(enc, "d") != 3:
        raise CheckpointError("encoding does not match the run's architecture")
    bm = _at(j, "b_matrix")
    if len(bm) != 3 * arch.m:
        raise CheckpointError("encoding matrix size does not match spec")
    shapes = _layer_shapes(arch)
    hidden = _at(j, "hidden")
    if len(hidden) != len(shapes) - 2:
        raise CheckpointError("hidden layer count does not match the run's architecture")
    parts = []
    for lj, shape in zip(list(hidden) + [_at(j, "head_material"), _at(j, "head_weight")], shapes):
        w, b = _layer_from_json(lj, shape)
        parts += [w, b]
    return np.array([x for p in parts for x in p], dtype=np.float64), np.array(bm, dtype=np.float64)


# --------------------------------------------------------------- run state
def state_to_json(st: EvolutionState) -> dict:
    """to_json(EvolutionState) (serialize.hpp:214-233)."""
    arch = st.config.arch
    pop = st.population()
    best_f, best_p = st.best()
    bm_best = None
    if best_p is not None:
        # best_genome carries its own B matrix: the device keeps it beside the params
        bm_best = st._best_bmat()
    return {"config": evolution_config_to_json(st.config), "params": hyper_params_to_json(st.params),
            "population": [{"genome": genome_to_json(pop["params"][a], pop["bmat"][a], arch),
                            "fitness": float(pop["fitness"][a]), "evaluated": bool(pop["evaluated"][a])}
                           for a in range(st.config.population)],
            "history": [report_to_json(r) for r in st.history], "generation": int(st.generation),
            "best_fitness": float(best_f), "rng": st.rng_state(),
            "best_genome": None if best_p is None else genome_to_json(best_p, bm_best, arch)}


def state_from_json(j: dict, ctx: Optional[Context] = None) -> EvolutionState:
    """evolution_state_from_json (serialize.hpp:235-262) into a device state."""
    cfg = evolution_config_from_json(_at(j, "config"))
    popj = _at(j, "population")
    if len(popj) != cfg.population:
        raise CheckpointError("population size does not match the config")
    st = EvolutionState(cfg, ctx)
    arch = cfg.arch
    n = param_count(arch)
    params = np.zeros((cfg.population, n))
    bmat = np.zeros((cfg.population, 3 * arch.m))
    fitness = np.zeros(cfg.population)
    evaluated = np.zeros(cfg.population, np.uint8)
    for a, ind in enumerate(popj):
        params[a], bmat[a] = genome_from_json(_at(ind, "genome"), arch)
        fitness[a] = _num(ind, "fitness")
        evaluated[a] = _bool(ind, "evaluated")
    st.set_population(params, bmat, fitness, evaluated)  # grids: decoded again next generation
    st.params = hyper_params_from_json(_at(j, "params"))
    st.history = [report_from_json(r) for r in _at(j, "history")]
    best_j = _at(j, "best_genome")
    best = None if best_j is None else genome_from_json(best_j, arch)
    st.set_progress(_int(j, "generation"), _num(j, "best_fitness"), best)
    rng = _at(j, "rng")
    if not isinstance(rng, str):
        raise CheckpointError("rng: expected a string")
    try:
        st.set_rng_state(rng)
    except ValueError as exc:
        raise CheckpointError(str(exc)) from exc
    return st


def wrap_payload(kind: str, payload: dict) -> dict:
    """wrap_payload (serialize.hpp:267-275)."""
    return {"magic": CHECKPOINT_MAGIC, "version": CHECKPOINT_VERSION, "kind": kind,
            "checksum": fnv1a64_hex(dumps(payload)), "payload": payload}


def unwrap_payload(j: Any, expected_kind: str) -> dict:
    """unwrap_payload (serialize.hpp:277-290)."""
    if not isinstance(j, dict) or j.get("magic", "") != CHECKPOINT_MAGIC:
        raise CheckpointError("not a voxevo checkpoint")
    if j.get("version", 0) != CHECKPOINT_VERSION:
        raise CheckpointError("unsupported checkpoint version")
    if j.get("kind", "") != expected_kind:
        raise CheckpointError("checkpoint kind mismatch: expected " + expected_kind)
    if "payload" not in j:
        raise CheckpointError("checkpoint has no payload")
    payload = j["payload"]
    if j.get("checksum", "") != fnv1a64_hex(dumps(payload)):
        raise CheckpointError("checkpoint checksum mismatch")
    return payload


def save_json_file(path: str, j: dict):
    """save_json_file (serialize.hpp:292-297): dump(2) + newline."""
    try:
        with open(path, "wb") as f:
            f.write((dumps(j, indent=2) + "\n").encode())
    except OSError as exc:
        raise CheckpointError("cannot open for writing: " + path) from exc


def load_json_file(path: str) -> Any:
    """load_json_file (serialize.hpp:299-305)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as exc:
        raise CheckpointError("cannot open: " + path) from exc
    try:
        return json.loads(data)
    except ValueError as exc:
        raise CheckpointError("invalid JSON: " + path) from exc


def save_run(path: str, st: EvolutionState):
    """save_run (serialize.hpp:307-309)."""
    save_json_file(path, wrap_payload("run", state_to_json(st)))


def load_run(path: str, ctx: Optional[Context] = None) -> EvolutionState:
    """load_run (serialize.hpp:311-313) -> a device-resident EvolutionState."""
    return state_from_json(unwrap_payload(load_json_file(path), "run"), ctx)


def save_genome(path: str, params: np.ndarray, bmat: np.ndarray, arch: Arch):
    """save_genome (serialize.hpp:315-317)."""
    save_json_file(path, wrap_payload("genome", genome_to_json(params, bmat, arch)))


def genome_arch(j: dict) -> Arch:
    """The architecture a genome JSON declares (encoding m / sigma, hidden
    layer widths) — what the reference's self-describing Genome carries."""
    enc = _at(j, "encoding")
    sigma = float(enc["sigma"]) if isinstance(enc, dict) and "sigma" in enc else 1.0
    widths = [_int(lj, "out") for lj in _at(j, "hidden")]
    try:
        return Arch.make(_int(enc, "m"), widths, sigma)
    except ValueError as e:
        raise CheckpointError(str(e)) from e


def load_genome(path: str, arch: Optional[Arch] = None) -> tuple:
    """load_genome (serialize.hpp:319-321) -> (flat params, b_matrix); with
    ``arch=None`` the architecture is read from the file and returned too:
    (flat params, b_matrix, arch)."""
    j = unwrap_payload(load_json_file(path), "genome")
    if arch is None:
        a = genome_arch(j)
        p, b = genome_from_json(j, a)
        return p, b, a
    return genome_from_json(j, arch)


def curves_csv(history: list) -> str:
    """curves_csv (serialize.hpp:327-343): wall_time written as 0."""
    rows = ["generation,mutation_rate,mutation_scale,crossover_rate,elite_fraction,"
            "best,mean,std,diversity,evaluations,wall_time\n"]
    for r in history:
        p = r.params
        vals = [p.mutation_rate, p.mutation_scale, p.crossover_rate, p.elite_fraction, r.best, r.mean, r.stddev,
                r.diversity]
        rows.append(str(int(r.generation)) + "".join("," + t for t in format_doubles(vals)) +
                    "," + str(int(r.evaluations)) + ",0\n")
    return "".join(rows)


def write_curves_csv(path: str, history: list):
    try:
        with open(path, "wb") as f:
            f.write(curves_csv(history).encode())
    except OSError as exc:
        raise CheckpointError("cannot open for writing: " + path) from exc
