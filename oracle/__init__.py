"""oracle — TEST INFRASTRUCTURE ONLY.  CPU checkers for the voxevo hot path.

Two interchangeable backends with the same API:

* ``restatement()``  -> ``liboracle.so``, our plain-C restatement
  (``oracle/voxevo_oracle.c``), every function citing the reference file:line
  it follows;
* ``reference()``    -> ``_ref/libvoxevo_ref.so``, the UNMODIFIED reference
  headers (``/root/reference/proj/include/voxevo``) compiled where they lie
  behind ``oracle/ref_shim.cpp``.

``tests/test_oracle_pinning.py`` proves the two bit-identical and pins both to
the golden vectors in ``tests/golden``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import this package.  The product (``paper_2405_00698_b200``) never does.
"""
from __future__ import annotations

import math
import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libvoxevo_ref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

DEFAULT_TABLE = np.array([2e3, 1e3, 1e4, 0.1, 0.25, np.pi, 0.1, 0.1])  # morphology.hpp:45-53
DEFAULT_PLANE = np.array([1e5, 0.1, 0.6, 1.0])  # morphology.hpp:124-129
DEFAULT_SIM = np.array([9.81, 1e-5, 2.0, 2.0, 1.0, 1.0])  # physics.hpp:16-22
DEFAULT_HYPER = np.array([0.1, 0.1, 0.4, 0.3, 1.0, 1.0, 1.0])  # evolution.hpp:22-27


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def sim6(gravity=9.81, dt=1e-5, duration=2.0, actuation_frequency=2.0, enable_gravity=True,
         enable_contact=True) -> np.ndarray:
    return np.array([gravity, dt, duration, actuation_frequency, float(enable_gravity), float(enable_contact)])


def _p(a, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class System:
    """A MassSpringSystem in flat arrays (morphology.hpp:110-135)."""
    pos: np.ndarray  # (nm, 3)
    vel: np.ndarray  # (nm, 3)
    mass: np.ndarray  # (nm,)
    si: np.ndarray  # (ns,) int32
    sj: np.ndarray
    k: np.ndarray
    rest0: np.ndarray
    zeta: np.ndarray
    has_act: np.ndarray  # uint8
    sign: np.ndarray
    amp: np.ndarray
    phase: np.ndarray
    plane: np.ndarray = field(default_factory=lambda: DEFAULT_PLANE.copy())

    @property
    def nm(self):
        return self.mass.shape[0]

    @property
    def ns(self):
        return self.k.shape[0]


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.pre = prefix
        self.path = path
        f = self._f
        vp = C.c_void_p
        f("rng_draws", None, [C.c_uint64, C.c_int64, vp])
        f("rng_uniform", None, [C.c_uint64, C.c_int64, vp])
        f("rng_normal", None, [C.c_uint64, C.c_int64, vp])
        f("rng_index", None, [C.c_uint64, C.c_int64, C.c_uint64, vp])
        f("rng_state", C.c_int64, [C.c_uint64, C.c_int64, C.c_char_p, C.c_int64])
        f("rng_draws_from_state", None, [C.c_char_p, C.c_int64, vp])
        f("param_count", C.c_int64, [C.c_int, C.c_int, vp])
        f("sample_genome", None, [C.c_int, C.c_double, C.c_int, vp, C.c_uint64, vp, vp])
        f("gaussian_encode", None, [vp, vp, C.c_int, vp])
        f("forward", None, [C.c_int, C.c_int, vp, vp, vp, vp, vp, vp])
        f("decode", None, [C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp])
        f("largest_component", None, [C.c_int, C.c_int, C.c_int, vp, vp])
        f("bench_robot", None, [C.c_int, vp, vp])
        f("build", vp, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp])
        f("sys_make", vp, [C.c_int, C.c_int] + [vp] * 13)
        f("sys_sizes", None, [vp, vp, vp])
        f("sys_export", None, [vp] * 13)
        f("sys_free", None, [vp])
        f("sys_workspace", None, [vp] * 9)
        f("sys_step", C.c_int64, [vp, vp, C.c_int64, C.c_int64, vp, vp, vp])
        f("center_of_mass", None, [vp, vp])
        f("evaluate_fitness", C.c_double, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp])
        f("population_diversity", C.c_double, [C.c_int, C.c_int, vp])
        f("elite_count", C.c_int, [C.c_double, C.c_int])
        f("hyper_clamp", None, [vp])
        f("evo_init", vp, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_double, C.c_int,
                           C.c_int, C.c_uint64, vp, vp, vp, vp])
        f("evo_free", None, [vp])
        f("evo_generation", None, [vp, vp])
        f("evo_get_population", None, [vp] * 7)
        f("evo_set_population", None, [vp] * 7)
        f("evo_rng_state", C.c_int64, [vp, C.c_char_p, C.c_int64])
        f("evo_set_rng_state", None, [vp, C.c_char_p])
        f("evo_get_params", None, [vp, vp])
        f("evo_set_params", None, [vp, vp])
        f("evo_best", C.c_int, [vp, vp, vp])
        if prefix == "ref_":
            f("simulate", C.c_int64, [vp, vp, vp, vp, C.c_int64, C.c_int])
            f("run_bench", None, [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_double, vp])
            f("evaluate_batch", C.c_double, [C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int, vp,
                                             vp])
            f("evo_set_threads", None, [vp, C.c_int])
            f("evo_generation_timed", C.c_double, [vp, vp, vp])
            f("evo_generation_advised", C.c_int, [vp, vp, vp])
            f("evo_pending_fitness", None, [vp, vp])
        else:
            f("simulate", None, [vp, vp, vp])

    def _f(self, name, restype, argtypes):
        fn = getattr(self.lib, self.pre + name)
        fn.restype = restype
        fn.argtypes = argtypes
        setattr(self, "_" + name, fn)

    # ---------------------------------------------------------------- rng
    def rng_draws(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._rng_draws(seed, n, out.ctypes.data)
        return out

    def rng_uniform(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n)
        self._rng_uniform(seed, n, out.ctypes.data)
        return out

    def rng_normal(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n)
        self._rng_normal(seed, n, out.ctypes.data)
        return out

    def rng_index(self, seed: int, n: int, rng: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._rng_index(seed, n, rng, out.ctypes.data)
        return out

    def rng_state(self, seed: int, skip: int) -> str:
        n = self._rng_state(seed, skip, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._rng_state(seed, skip, buf, n + 1)
        return buf.value.decode()

    def rng_draws_from_state(self, state: str, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._rng_draws_from_state(state.encode(), n, out.ctypes.data)
        return out

    # -------------------------------------------------------------- genome
    @staticmethod
    def _w(widths):
        return np.ascontiguousarray(widths, dtype=np.int32)

    def param_count(self, m: int, widths) -> int:
        w = self._w(widths)
        return int(self._param_count(m, len(w), w.ctypes.data))

    def sample_genome(self, m: int, widths, seed: int, sigma: float = 1.0):
        w = self._w(widths)
        params = np.zeros(self.param_count(m, widths))
        bmat = np.zeros(3 * m)
        self._sample_genome(m, sigma, len(w), w.ctypes.data, seed, params.ctypes.data, bmat.ctypes.data)
        return params, bmat

    def gaussian_encode(self, v, bmat, m: int):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(2 * m)
        self._gaussian_encode(v.ctypes.data, np.ascontiguousarray(bmat).ctypes.data, m, out.ctypes.data)
        return out

    def forward(self, m, widths, params, bmat, v):
        w = self._w(widths)
        v = np.ascontiguousarray(v, np.float64)
        probs = np.zeros(5)
        wt = np.zeros(1)
        self._forward(m, len(w), w.ctypes.data, np.ascontiguousarray(params).ctypes.data,
                      np.ascontiguousarray(bmat).ctypes.data, v.ctypes.data, probs.ctypes.data, wt.ctypes.data)
        return probs, float(wt[0])

    def decode(self, m, widths, params, bmat, w, h, d):
        wd = self._w(widths)
        mat = np.zeros(w * h * d, np.uint8)
        wt = np.zeros(w * h * d)
        self._decode(m, len(wd), wd.ctypes.data, np.ascontiguousarray(params).ctypes.data,
                     np.ascontiguousarray(bmat).ctypes.data, w, h, d, mat.ctypes.data, wt.ctypes.data)
        return mat, wt

    def largest_component(self, mat, w, h, d):
        mat = np.ascontiguousarray(mat, np.uint8)
        out = np.zeros_like(mat)
        self._largest_component(w, h, d, mat.ctypes.data, out.ctypes.data)
        return out

    def bench_robot(self, n):
        mat = np.zeros(n ** 3, np.uint8)
        wt = np.zeros(n ** 3)
        self._bench_robot(n, mat.ctypes.data, wt.ctypes.data)
        return mat, wt

    # ------------------------------------------------------------- systems
    def _export(self, h) -> System:
        nm = C.c_int()
        ns = C.c_int()
        self._sys_sizes(h, C.byref(nm), C.byref(ns))
        nm, ns = nm.value, ns.value
        s = System(pos=np.zeros((nm, 3)), vel=np.zeros((nm, 3)), mass=np.zeros(nm), si=np.zeros(ns, np.int32),
                   sj=np.zeros(ns, np.int32), k=np.zeros(ns), rest0=np.zeros(ns), zeta=np.zeros(ns),
                   has_act=np.zeros(ns, np.uint8), sign=np.zeros(ns), amp=np.zeros(ns), phase=np.zeros(ns))
        self._sys_export(h, s.pos.ctypes.data, s.vel.ctypes.data, s.mass.ctypes.data, s.si.ctypes.data,
                         s.sj.ctypes.data, s.k.ctypes.data, s.rest0.ctypes.data, s.zeta.ctypes.data,
                         s.has_act.ctypes.data, s.sign.ctypes.data, s.amp.ctypes.data, s.phase.ctypes.data)
        return s

    def build(self, mat, wt, w, h, d, table=None, plane=None):
        """build_mass_spring (morphology.hpp:217-299); None for an empty grid."""
        mat = np.ascontiguousarray(mat, np.uint8)
        wt = np.ascontiguousarray(wt, np.float64)
        table = DEFAULT_TABLE if table is None else np.ascontiguousarray(table, np.float64)
        plane = DEFAULT_PLANE if plane is None else np.ascontiguousarray(plane, np.float64)
        h_ = self._build(w, h, d, mat.ctypes.data, wt.ctypes.data, table.ctypes.data, plane.ctypes.data)
        if not h_:
            return None
        try:
            s = self._export(h_)
        finally:
            self._sys_free(h_)
        s.plane = plane.copy()
        return s

    def _make(self, s: System):
        c = np.ascontiguousarray
        arrs = [c(s.pos, np.float64), c(s.vel, np.float64), c(s.mass, np.float64), c(s.si, np.int32),
                c(s.sj, np.int32), c(s.k, np.float64), c(s.rest0, np.float64), c(s.zeta, np.float64),
                c(s.has_act, np.uint8), c(s.sign, np.float64), c(s.amp, np.float64), c(s.phase, np.float64),
                c(s.plane, np.float64)]
        h = self._sys_make(s.nm, s.ns, *[a.ctypes.data for a in arrs])
        return h

    def workspace(self, s: System) -> dict:
        h = self._make(s)
        try:
            ns, nm = s.ns, s.nm
            out = dict(damp_coef=np.zeros(ns), amp_rest=np.zeros(ns), sin_phase=np.zeros(ns), cos_phase=np.zeros(ns),
                       ground_damp=np.zeros(nm), inc_off=np.zeros(nm + 1, np.int32),
                       inc_spring=np.zeros(2 * ns, np.int32), inc_sign=np.zeros(2 * ns))
            self._sys_workspace(h, *[out[k].ctypes.data for k in
                                     ("damp_coef", "amp_rest", "sin_phase", "cos_phase", "ground_damp", "inc_off",
                                      "inc_spring", "inc_sign")])
        finally:
            self._sys_free(h)
        return out

    def step(self, s: System, sim=None, k0: int = 0, nsteps: int = 1):
        """Run step() (physics.hpp:191-264) nsteps times from k0; returns
        (new System, ok_steps, steps_called, spring_updates, max_speed_sq)."""
        sim = DEFAULT_SIM if sim is None else np.ascontiguousarray(sim, np.float64)
        h = self._make(s)
        try:
            called = C.c_int64()
            upd = C.c_uint64()
            msq = C.c_double()
            ok = self._sys_step(h, sim.ctypes.data, k0, nsteps, C.byref(called), C.byref(upd), C.byref(msq))
            out = self._export(h)
            out.plane = s.plane.copy()
        finally:
            self._sys_free(h)
        return out, int(ok), int(called.value), int(upd.value), float(msq.value)

    def simulate(self, s: System, sim=None, stride=None) -> dict:
        """simulate (physics.hpp:287-311); with ``stride`` (reference library
        only) also the TrajectorySample dump as an (rows, 4) array."""
        sim = DEFAULT_SIM if sim is None else np.ascontiguousarray(sim, np.float64)
        h = self._make(s)
        summ = np.zeros(9)
        dump = None
        try:
            if stride is not None:
                if self.pre != "ref_":
                    raise RuntimeError("the trajectory dump needs the reference library (oracle/_ref)")
                n_steps = int(math.floor(sim[2] / sim[1] + 0.5))  # llround
                cap = (-(-n_steps // stride) if stride > 0 else 0) + 1
                dump = np.zeros((cap, 4))
                rows = self._simulate(h, sim.ctypes.data, summ.ctypes.data, dump.ctypes.data, cap, int(stride))
                dump = dump[:min(int(rows), cap)].copy()
            elif self.pre == "ref_":
                self._simulate(h, sim.ctypes.data, summ.ctypes.data, None, 0, 0)
            else:
                self._simulate(h, sim.ctypes.data, summ.ctypes.data)
        finally:
            self._sys_free(h)
        out = dict(com_start=summ[0:3].copy(), com_end=summ[3:6].copy(), horizontal_displacement=float(summ[6]),
                   max_speed=float(summ[7]), diverged=bool(summ[8] != 0.0))
        if dump is not None:
            out["dump"] = dump
        return out

    def evaluate_fitness(self, mat, wt, w, h, d, table=None, plane=None, sim=None) -> float:
        mat = np.ascontiguousarray(mat, np.uint8)
        wt = np.ascontiguousarray(wt, np.float64)
        table = DEFAULT_TABLE if table is None else np.ascontiguousarray(table, np.float64)
        plane = DEFAULT_PLANE if plane is None else np.ascontiguousarray(plane, np.float64)
        sim = DEFAULT_SIM if sim is None else np.ascontiguousarray(sim, np.float64)
        return float(self._evaluate_fitness(w, h, d, mat.ctypes.data, wt.ctypes.data, table.ctypes.data,
                                            plane.ctypes.data, sim.ctypes.data))

    def population_diversity(self, mats) -> float:
        mats = np.ascontiguousarray(mats, np.uint8)
        return float(self._population_diversity(mats.shape[0], mats.shape[1], mats.ctypes.data))

    def elite_count(self, ef: float, P: int) -> int:
        return int(self._elite_count(ef, P))

    def hyper_clamp(self, h7):
        h = np.ascontiguousarray(h7, np.float64).copy()
        self._hyper_clamp(h.ctypes.data)
        return h

    # ----------------------------------------------------------- evolution
    def evo(self, **kw) -> "Evo":
        return Evo(self, **kw)


class Evo:
    """EvolutionState + evolve_generation (evolution.hpp:177-293), advisor off."""

    def __init__(self, lib: _Lib, population=30, generations=100, grid=(5, 5, 5), hidden=(64, 64), m=32, sigma=1.0,
                 tournament=3, threads=1, seed=0, hyper=None, table=None, plane=None, sim=None):
        self.lib = lib
        self.P = population
        self.grid = tuple(grid)
        self.cells = grid[0] * grid[1] * grid[2]
        self.m = m
        self.hidden = tuple(hidden)
        self.np = lib.param_count(m, hidden)
        w = np.ascontiguousarray(hidden, np.int32)
        hyper = DEFAULT_HYPER if hyper is None else np.ascontiguousarray(hyper, np.float64)
        table = DEFAULT_TABLE if table is None else np.ascontiguousarray(table, np.float64)
        plane = DEFAULT_PLANE if plane is None else np.ascontiguousarray(plane, np.float64)
        sim = DEFAULT_SIM if sim is None else np.ascontiguousarray(sim, np.float64)
        self.h = lib._evo_init(population, generations, grid[0], grid[1], grid[2], len(w), w.ctypes.data, m, sigma,
                               tournament, threads, seed, hyper.ctypes.data, table.ctypes.data, plane.ctypes.data,
                               sim.ctypes.data)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib._evo_free(self.h)
            self.h = None

    def generation(self) -> dict:
        rep = np.zeros(14)
        self.lib._evo_generation(self.h, rep.ctypes.data)
        return dict(generation=int(rep[0]), best=float(rep[1]), mean=float(rep[2]), stddev=float(rep[3]),
                    diversity=float(rep[4]), evaluations=int(rep[5]), wall_time=float(rep[6]),
                    params=rep[7:14].copy())

    def generation_advised(self, adv4=None) -> dict:
        """evolve_generation with the reference's own ScriptedAdvisor
        (advisor.hpp:30-55) in the loop; adv4 = (diversity_floor,
        stagnation_eps, mutation_boost, crossover_boost) or None for defaults."""
        rep = np.zeros(14)
        a = None if adv4 is None else np.ascontiguousarray(adv4, np.float64)
        if not self.lib._evo_generation_advised(self.h, rep.ctypes.data, None if a is None else a.ctypes.data):
            raise RuntimeError("reference built without nlohmann/json: ScriptedAdvisor unavailable")
        return dict(generation=int(rep[0]), best=float(rep[1]), mean=float(rep[2]), stddev=float(rep[3]),
                    diversity=float(rep[4]), evaluations=int(rep[5]), wall_time=float(rep[6]),
                    params=rep[7:14].copy())

    def pending_fitness(self) -> np.ndarray:
        """The fitness the next evolve_generation computes for each individual
        without a cached score (NaN for the others)."""
        out = np.zeros(self.P)
        self.lib._evo_pending_fitness(self.h, out.ctypes.data)
        return out

    def generation_timed(self):
        """(report, seconds of evolve_generation alone, exact spring updates it performed)."""
        rep = np.zeros(14)
        upd = np.zeros(1, np.uint64)
        secs = self.lib._evo_generation_timed(self.h, rep.ctypes.data, upd.ctypes.data)
        return dict(generation=int(rep[0]), best=float(rep[1]), mean=float(rep[2]), stddev=float(rep[3]),
                    diversity=float(rep[4]), evaluations=int(rep[5]), wall_time=float(rep[6]),
                    params=rep[7:14].copy()), float(secs), int(upd[0])

    def population(self) -> dict:
        P, np_, cells = self.P, self.np, self.cells
        out = dict(params=np.zeros((P, np_)), bmat=np.zeros((P, 3 * self.m)), fitness=np.zeros(P),
                   evaluated=np.zeros(P, np.uint8), grids=np.zeros((P, cells), np.uint8),
                   grid_w=np.zeros((P, cells)))
        self.lib._evo_get_population(self.h, *[out[k].ctypes.data for k in
                                               ("params", "bmat", "fitness", "evaluated", "grids", "grid_w")])
        return out

    def set_population(self, params, bmat, fitness=None, evaluated=None, grids=None, grid_w=None):
        c = np.ascontiguousarray
        arrs = [c(params, np.float64), c(bmat, np.float64),
                None if fitness is None else c(fitness, np.float64),
                None if evaluated is None else c(evaluated, np.uint8),
                None if grids is None else c(grids, np.uint8),
                None if grid_w is None else c(grid_w, np.float64)]
        self._keep = arrs
        self.lib._evo_set_population(self.h, *[None if a is None else a.ctypes.data for a in arrs])

    def rng_state(self) -> str:
        n = self.lib._evo_rng_state(self.h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib._evo_rng_state(self.h, buf, n + 1)
        return buf.value.decode()

    def set_rng_state(self, s: str):
        self.lib._evo_set_rng_state(self.h, s.encode())

    def params(self):
        h = np.zeros(7)
        self.lib._evo_get_params(self.h, h.ctypes.data)
        return h

    def set_params(self, h7):
        h = np.ascontiguousarray(h7, np.float64)
        self.lib._evo_set_params(self.h, h.ctypes.data)

    def best(self):
        bf = C.c_double()
        bp = np.zeros(self.np)
        has = self.lib._evo_best(self.h, C.byref(bf), bp.ctypes.data)
        return float(bf.value), (bp if has else None)


_cache: dict = {}


def restatement() -> _Lib:
    if "orc" not in _cache:
        _cache["orc"] = _Lib(ORC_SO, "orc_")
    return _cache["orc"]


def reference() -> _Lib:
    if "ref" not in _cache:
        _cache["ref"] = _Lib(REF_SO, "ref_")
    return _cache["ref"]


def have_reference() -> bool:
    return os.path.exists(REF_SO)


REF_IO_SO = os.path.join(HERE, "_ref", "libvoxevo_ref_io.so")


class RefIO:
    """The reference's serialize.hpp (checkpoints, curves) and its JSON
    library's number printing, behind oracle/ref_io_shim.cpp."""

    def __init__(self, path: str = REF_IO_SO):
        lib = C.CDLL(path)
        i64, vp, cp = C.c_int64, C.c_void_p, C.c_char_p
        lib.ref_io_last_error.restype = cp
        lib.ref_io_dump_doubles.restype = i64
        lib.ref_io_dump_doubles.argtypes = [vp, i64, cp, i64]
        lib.ref_io_fnv_hex.restype = i64
        lib.ref_io_fnv_hex.argtypes = [cp, cp, i64]
        lib.ref_io_run_and_save.restype = C.c_int
        lib.ref_io_run_and_save.argtypes = [cp, C.c_int, cp]
        lib.ref_io_resume.restype = C.c_int
        lib.ref_io_resume.argtypes = [cp, C.c_int, cp]
        lib.ref_io_curves_csv.restype = i64
        lib.ref_io_curves_csv.argtypes = [cp, cp, i64]
        lib.ref_io_run_advised.restype = C.c_int
        lib.ref_io_run_advised.argtypes = [cp, C.c_int, vp, vp, cp, i64]
        self.lib = lib

    def _text(self, fn, *args) -> str:
        n = fn(*args, None, 0)
        if n < 0:
            raise RuntimeError(self.lib.ref_io_last_error().decode())
        buf = C.create_string_buffer(n + 1)
        fn(*args, buf, n + 1)
        return buf.raw[:n].decode()

    def dump_doubles(self, v: np.ndarray) -> list:
        v = np.ascontiguousarray(v, np.float64)
        return self._text(self.lib.ref_io_dump_doubles, v.ctypes.data, v.size)[1:-1].split(",")

    def fnv_hex(self, s: str) -> str:
        return self._text(self.lib.ref_io_fnv_hex, s.encode())

    def run_and_save(self, config_json: str, gens: int, path: str):
        if self.lib.ref_io_run_and_save(config_json.encode(), gens, path.encode()) != 0:
            raise RuntimeError(self.lib.ref_io_last_error().decode())

    def resume(self, in_path: str, gens: int, out_path: str):
        if self.lib.ref_io_resume(in_path.encode(), gens, out_path.encode()) != 0:
            raise RuntimeError(self.lib.ref_io_last_error().decode())

    def curves_csv(self, path: str) -> str:
        return self._text(self.lib.ref_io_curves_csv, path.encode())

    def run_advised(self, config_json: str, gens: int, adv4=None):
        """init_evolution + gens x evolve_generation with the reference's own
        ScriptedAdvisor (advisor.hpp:30-55).  Returns (history rows [gens][13]:
        generation, best, mean, stddev, diversity, evaluations, params[7]; the
        final Rng state text)."""
        hist = np.zeros((gens, 13))
        a = None if adv4 is None else np.ascontiguousarray(adv4, np.float64)
        buf = C.create_string_buffer(1 << 16)
        if self.lib.ref_io_run_advised(config_json.encode(), gens, None if a is None else a.ctypes.data,
                                       hist.ctypes.data, buf, len(buf)) != 0:
            raise RuntimeError(self.lib.ref_io_last_error().decode())
        return hist, buf.value.decode()


def have_reference_io() -> bool:
    return os.path.exists(REF_IO_SO)


def reference_io() -> RefIO:
    if "io" not in _cache:
        _cache["io"] = RefIO()
    return _cache["io"]


# --------------------------------------------------------------------------
# Hand-built systems used by the reference's own physics tests
# (test_physics.cpp:13-27, acceptance_main.cpp:77-92).
def dumbbell(mass: float, k: float, rest: float, separation: float, damping_ratio: float = 0.0) -> System:
    return System(pos=np.array([[0.0, 0.0, 1.0], [separation, 0.0, 1.0]]), vel=np.zeros((2, 3)),
                  mass=np.array([mass, mass]), si=np.array([0], np.int32), sj=np.array([1], np.int32),
                  k=np.array([k]), rest0=np.array([rest]), zeta=np.array([damping_ratio]),
                  has_act=np.zeros(1, np.uint8), sign=np.zeros(1), amp=np.zeros(1), phase=np.zeros(1))
