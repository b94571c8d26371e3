"""paper_2405_00698_b200 — B200-native (sm_100a) voxevo hot path.

Python mirror of the reference's ``voxevo::`` API for the data-parallel path
(decode -> largest_component -> build_mass_spring -> simulate ->
evaluate_fitness -> evolve_generation, plus run_bench), implemented by the
C-ABI CUDA library ``_lib/libvoxevo_b200.so`` (``include/voxevo_b200.h``).

There is no CPU fallback: every entry point runs on the GPU through the
library, and importing the bindings raises if the library is missing or no
sm_100 device is usable.  Names, argument meaning and error behaviour follow
the reference (citations are to /root/reference/proj/include/voxevo/):
invalid arguments raise ``ValueError`` (std::invalid_argument), an empty grid
raises ``EmptyRobot`` (morphology.hpp:17-19), numerical divergence is reported
as data (``TrajectorySummary.diverged``, fitness 0).
"""
from __future__ import annotations

import math
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libvoxevo_b200.so")

VX_OK, VX_EINVAL, VX_ECUDA, VX_EOOM, VX_EEMPTY, VX_ESHAPE, VX_ESTATE, VX_ENODEV, VX_ENCCL = range(9)
NMAT = 5
MAX_HIDDEN = 8

# Material enum (morphology.hpp:21-27)
EMPTY, MUSCLE_EXPAND, MUSCLE_CONTRACT, SOFT_TISSUE, HARD_BONE = range(5)


class VoxevoError(RuntimeError):
    pass


class EmptyRobot(VoxevoError):
    """empty_robot (morphology.hpp:17-19)."""


class ShapeMismatch(VoxevoError):
    """shape_mismatch (genome.hpp:19-21)."""


class DeviceUnavailable(VoxevoError):
    pass


# ----------------------------------------------------------------- C structs
class Arch(C.Structure):
    """EncodingSpec + hidden widths (genome.hpp:25-35)."""
    _fields_ = [("m", C.c_int32), ("n_hidden", C.c_int32), ("hidden", C.c_int32 * MAX_HIDDEN),
                ("sigma", C.c_double)]

    @classmethod
    def make(cls, m: int = 32, hidden: Sequence[int] = (64, 64), sigma: float = 1.0) -> "Arch":
        if len(hidden) > MAX_HIDDEN:
            raise ValueError("at most %d hidden layers" % MAX_HIDDEN)
        a = cls()
        a.m = m
        a.n_hidden = len(hidden)
        for i, w in enumerate(hidden):
            a.hidden[i] = w
        a.sigma = sigma
        return a

    @property
    def widths(self):
        return [self.hidden[i] for i in range(self.n_hidden)]


class MaterialTable(C.Structure):
    """MaterialTable (morphology.hpp:45-65)."""
    _fields_ = [(n, C.c_double) for n in ("k_muscle", "k_soft", "k_bone", "damping_ratio", "amp_max", "phase_max",
                                          "voxel_edge", "mass_per_vertex")]

    def __init__(self, **kw):
        super().__init__(2e3, 1e3, 1e4, 0.1, 0.25, np.pi, 0.1, 0.1)
        for k, v in kw.items():
            setattr(self, k, v)

    def as_array(self):
        return np.array([getattr(self, f) for f, _ in self._fields_])


class GroundPlane(C.Structure):
    """GroundPlane (morphology.hpp:124-129)."""
    _fields_ = [(n, C.c_double) for n in ("k", "damping_ratio", "mu_static", "mu_kinetic")]

    def __init__(self, **kw):
        super().__init__(1e5, 0.1, 0.6, 1.0)
        for k, v in kw.items():
            setattr(self, k, v)

    def as_array(self):
        return np.array([getattr(self, f) for f, _ in self._fields_])


class SimConfig(C.Structure):
    """SimConfig (physics.hpp:16-29)."""
    _fields_ = [("gravity", C.c_double), ("dt", C.c_double), ("duration", C.c_double),
                ("actuation_frequency", C.c_double), ("enable_gravity", C.c_int32), ("enable_contact", C.c_int32)]

    def __init__(self, **kw):
        super().__init__(9.81, 1e-5, 2.0, 2.0, 1, 1)
        for k, v in kw.items():
            setattr(self, k, int(v) if k.startswith("enable") else v)

    def validate(self):
        if not self.dt > 0.0:
            raise ValueError("SimConfig: dt must be > 0")
        if not self.duration >= 0.0:
            raise ValueError("SimConfig: duration must be >= 0")
        if not self.actuation_frequency > 0.0:
            raise ValueError("SimConfig: frequency must be > 0")

    def as_array(self):
        return np.array([self.gravity, self.dt, self.duration, self.actuation_frequency,
                         float(self.enable_gravity), float(self.enable_contact)])


class TrajectorySummary(C.Structure):
    """TrajectorySummary (physics.hpp:31-37) + exact work audit."""
    _fields_ = [("com_start", C.c_double * 3), ("com_end", C.c_double * 3), ("horizontal_displacement", C.c_double),
                ("max_speed", C.c_double), ("diverged", C.c_int32), ("status", C.c_int32), ("steps", C.c_int64),
                ("spring_updates", C.c_uint64)]


class HyperParams(C.Structure):
    """HyperParams (evolution.hpp:22-38)."""
    _fields_ = [("mutation_rate", C.c_double), ("mutation_scale", C.c_double), ("crossover_rate", C.c_double),
                ("elite_fraction", C.c_double), ("material_multipliers", C.c_double * 3)]

    def __init__(self, **kw):
        super().__init__(0.1, 0.1, 0.4, 0.3, (C.c_double * 3)(1.0, 1.0, 1.0))
        for k, v in kw.items():
            if k == "material_multipliers":
                self.material_multipliers = (C.c_double * 3)(*v)
            else:
                setattr(self, k, v)

    def clamp(self):
        _lib().vx_hyper_clamp(C.byref(self))
        return self

    def as_array(self):
        return np.array([self.mutation_rate, self.mutation_scale, self.crossover_rate, self.elite_fraction,
                         *self.material_multipliers])

    def copy(self):
        h = HyperParams()
        C.memmove(C.byref(h), C.byref(self), C.sizeof(self))
        return h


class EvolutionConfig(C.Structure):
    """EvolutionConfig (evolution.hpp:40-64)."""
    _fields_ = [("population", C.c_int32), ("generations", C.c_int32), ("grid_w", C.c_int32), ("grid_h", C.c_int32),
                ("grid_d", C.c_int32), ("tournament_size", C.c_int32), ("threads", C.c_int32), ("seed", C.c_uint64),
                ("arch", Arch), ("initial_params", HyperParams), ("materials", MaterialTable),
                ("plane", GroundPlane), ("sim", SimConfig)]

    def __init__(self, **kw):
        super().__init__()
        _lib().vx_default_evo_config(C.byref(self))
        for k, v in kw.items():
            if k == "grid":
                self.grid_w, self.grid_h, self.grid_d = v
            elif k == "hidden_widths":
                self.arch = Arch.make(self.arch.m, v, self.arch.sigma)
            elif k in ("m", "sigma"):
                setattr(self.arch, k, v)
            else:
                setattr(self, k, v)


class GenerationReport(C.Structure):
    """GenerationReport (evolution.hpp:75-84) + exact spring-update count."""
    _fields_ = [("generation", C.c_int32), ("evaluations", C.c_int32), ("params", HyperParams), ("best", C.c_double),
                ("mean", C.c_double), ("stddev", C.c_double), ("diversity", C.c_double), ("wall_time", C.c_double),
                ("spring_updates", C.c_uint64)]


# ------------------------------------------------------------------- loading
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(
                f"{LIB_PATH} is missing: build it with `make -C {HERE}` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        _declare(lib)
        if lib.vx_abi_version() != 3:
            raise DeviceUnavailable("libvoxevo_b200 ABI mismatch")
        _LIB = lib
    return _LIB


def _declare(lib):
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    P = C.POINTER
    sigs = {
        "vx_abi_version": (i32, []),
        "vx_last_error": (C.c_char_p, []),
        "vx_default_evo_config": (None, [P(EvolutionConfig)]),
        "vx_param_count": (i64, [P(Arch)]),
        "vx_elite_count": (i32, [dbl, i32]),
        "vx_hyper_clamp": (None, [P(HyperParams)]),
        "vx_create": (i32, [i32, P(vp)]),
        "vx_destroy": (i32, [vp]),
        "vx_set_stream": (i32, [vp, vp]),
        "vx_get_stream": (vp, [vp]),
        "vx_synchronize": (i32, [vp]),
        "vx_launch_count": (u64, [vp]),
        "vx_last_integrator": (i32, [vp]),
        "vx_set_filler": (i32, [vp, i32]),
        "vx_last_filler_ctas": (i32, [vp]),
        "vx_device_info": (i32, [vp, P(i32), P(i32), C.c_char_p, i32]),
        "vx_sample_genomes_dev": (i32, [vp, P(Arch), i32, vp, vp, vp]),
        "vx_decode_dev": (i32, [vp, P(Arch), i32, vp, vp, i32, i32, i32, vp, vp, vp]),
        "vx_decode": (i32, [vp, P(Arch), i32, vp, vp, i32, i32, i32, vp, vp]),
        "vx_decode_refined": (i32, [vp, P(C.c_int64)]),
        "vx_largest_component_dev": (i32, [vp, i32, i32, i32, i32, vp, vp]),
        "vx_largest_component": (i32, [vp, i32, i32, i32, i32, vp, vp]),
        "vx_batch_build_dev": (i32, [vp, i32, i32, i32, i32, vp, vp, P(MaterialTable), P(GroundPlane), P(vp)]),
        "vx_batch_build": (i32, [vp, i32, i32, i32, i32, vp, vp, P(MaterialTable), P(GroundPlane), P(vp)]),
        "vx_batch_upload": (i32, [vp, i32, vp, vp] + [vp] * 12 + [P(GroundPlane), P(vp)]),
        "vx_batch_free": (i32, [vp]),
        "vx_batch_count": (i32, [vp]),
        "vx_batch_offsets": (i32, [vp, vp, vp]),
        "vx_batch_download": (i32, [vp] * 13),
        "vx_batch_set_state": (i32, [vp, vp, vp]),
        "vx_batch_workspace": (i32, [vp] * 9),
        "vx_batch_override_phase": (i32, [vp, vp, vp]),
        "vx_batch_step": (i32, [vp, vp, P(SimConfig), i64, i64, vp]),
        "vx_batch_simulate": (i32, [vp, vp, P(SimConfig), vp]),
        "vx_batch_step_at": (i32, [vp, vp, P(SimConfig), dbl, vp]),
        "vx_batch_simulate_dev": (i32, [vp, vp, P(SimConfig), vp]),
        "vx_batch_simulate_dump": (i32, [vp, vp, P(SimConfig), i32, i64, vp, vp, vp]),
        "vx_evaluate_dev": (i32, [vp, i32, i32, i32, i32, vp, vp, P(MaterialTable), P(GroundPlane), P(SimConfig), vp,
                                 i32, vp, vp]),
        "vx_evaluate": (i32, [vp, i32, i32, i32, i32, vp, vp, P(MaterialTable), P(GroundPlane), P(SimConfig), vp,
                             vp]),
        "vx_population_diversity_dev": (i32, [vp, i32, i32, vp, vp]),
        "vx_population_diversity": (i32, [vp, i32, i32, vp, P(dbl)]),
        "vx_material_histogram_dev": (i32, [vp, i32, i32, vp, vp, i32]),
        "vx_diversity_from_histogram_dev": (i32, [vp, i32, i32, vp, vp]),
        "vx_evo_create": (i32, [vp, P(EvolutionConfig), P(vp)]),
        "vx_evo_free": (i32, [vp]),
        "vx_evo_generation": (i32, [vp, P(GenerationReport)]),
        "vx_evo_begin": (i32, [vp, i32, i32]),
        "vx_evo_exchange_buffer": (i32, [vp, P(vp), P(i64)]),
        "vx_evo_finish": (i32, [vp, P(GenerationReport)]),
        "vx_evo_set_exchange_buffer": (i32, [vp, vp]),
        "vx_evo_load_population_dev": (i32, [vp, vp, vp]),
        "vx_evo_get_population": (i32, [vp] * 7),
        "vx_evo_set_population": (i32, [vp] * 7),
        "vx_evo_population_dev": (i32, [vp, P(vp), P(vp), P(vp)]),
        "vx_evo_rng_state": (i64, [vp, C.c_char_p, i64]),
        "vx_evo_set_rng_state": (i32, [vp, C.c_char_p]),
        "vx_evo_get_params": (i32, [vp, P(HyperParams)]),
        "vx_evo_set_params": (i32, [vp, P(HyperParams)]),
        "vx_evo_generation_index": (i32, [vp]),
        "vx_evo_best": (i32, [vp, P(dbl), vp]),
        "vx_evo_best_genome": (i32, [vp, P(dbl), vp, vp]),
        "vx_evo_set_progress": (i32, [vp, i32, dbl, vp, vp]),
        "vx_run_bench": (i32, [vp, i32, i64, i32, dbl, vp]),
        "vx_timing_enable": (i32, [vp, i32]),
        "vx_integrator_timing": (i32, [vp, P(dbl), P(i64), i32]),
        "vx_fp64_peak": (i32, [vp, P(dbl)]),
        "vx_decode_timing": (i32, [vp, P(dbl), P(i64), i32]),
        "vx_dmma_peak": (i32, [vp, P(dbl)]),
        "vx_fastmath_check": (i32, [vp, i64, u64, vp]),
        "vx_format_doubles": (i64, [vp, i64, C.c_char, C.c_char_p, i64]),
        "vx_fnv1a64": (u64, [C.c_char_p, i64]),
        "vx_sample_genomes": (i32, [vp, P(Arch), i32, vp, vp, vp]),
        "vx_gaussian_encode": (i32, [vp, vp, i32, vp]),
        "vx_forward": (i32, [vp, P(Arch), i32, vp, vp, i32, vp, vp, vp]),
        "vx_rng_create": (i32, [u64, P(vp)]),
        "vx_rng_free": (None, [vp]),
        "vx_rng_next_u64": (u64, [vp]),
        "vx_rng_uniform01": (dbl, [vp]),
        "vx_rng_normal": (dbl, [vp]),
        "vx_rng_index": (u64, [vp, u64]),
        "vx_rng_state": (i64, [vp, C.c_char_p, i64]),
        "vx_rng_set_state": (i32, [vp, C.c_char_p]),
        "vx_crossover": (i32, [vp, i64, vp, vp, vp]),
        "vx_mutate": (i32, [vp, i64, vp, dbl, dbl]),
        "vx_tournament_select": (i32, [vp, i32, i32]),
        "vx_comm_available": (i32, []),
        "vx_comm_unique_id": (i32, [vp]),
        "vx_comm_create": (i32, [vp, i32, i32, vp, P(vp)]),
        "vx_comm_create_all": (i32, [i32, vp, vp]),
        "vx_comm_destroy": (i32, [vp]),
        "vx_comm_rank": (i32, [vp, P(i32), P(i32)]),
        "vx_comm_allreduce_sum_dev": (i32, [vp, vp, i64]),
        "vx_evo_set_comm": (i32, [vp, vp]),
        "vx_evo_set_exchange": (i32, [vp, i32, i32, vp, vp]),
        "vx_evo_generation_group": (i32, [i32, vp, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def exported_symbols() -> list:
    """The ABI entry points declared in include/voxevo_b200.h."""
    hdr = os.path.join(os.path.dirname(HERE), "include", "voxevo_b200.h")
    import re
    txt = open(hdr).read()
    return sorted(set(re.findall(r"^[a-z_0-9\* ]*?\b(vx_[a-z_0-9]+)\(", txt, re.M)))


def _check(st: int, what: str = ""):
    if st == VX_OK:
        return
    msg = (_lib().vx_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if st == VX_EINVAL:
        raise ValueError(text)
    if st == VX_EEMPTY:
        raise EmptyRobot(text)
    if st == VX_ESHAPE:
        raise ShapeMismatch(text)
    if st == VX_ENODEV:
        raise DeviceUnavailable(text)
    if st == VX_ENCCL:
        raise VoxevoError(f"NCCL: {text}")
    raise VoxevoError(f"status {st}: {text}")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def param_count(arch: Arch) -> int:
    """Genome::parameter_count (genome.hpp:83-87)."""
    n = _lib().vx_param_count(C.byref(arch))
    if n < 0:
        raise ValueError("invalid architecture")
    return int(n)


def elite_count(elite_fraction: float, population: int) -> int:
    """detail::elite_count (evolution.hpp:131-136)."""
    return int(_lib().vx_elite_count(elite_fraction, population))


# ------------------------------------------------------------------ context
class Context:
    """One per device: stream, scratch, launch counter (vx_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib().vx_create(device, C.byref(h)), "vx_create")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _lib().vx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: Optional[int]):
        _check(_lib().vx_set_stream(self.h, stream_handle), "vx_set_stream")

    def synchronize(self):
        _check(_lib().vx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(_lib().vx_launch_count(self.h))

    @property
    def last_integrator(self) -> str:
        """Kernel of the last integrator launch: generic | lattice | cluster | stream."""
        k = int(_lib().vx_last_integrator(self.h))
        return {0: "generic", 1: "lattice", 2: "cluster", 3: "stream"}.get(k, "none")

    def set_filler(self, mode: int):
        """10^3 cluster integrator's one-SM filler on the SMs no 4-CTA cluster
        can use: -1 from VX_FILLER (default on), 0 off, 1 on for large batches,
        2 on at any batch size."""
        _check(_lib().vx_set_filler(self.h, int(mode)), "vx_set_filler")

    @property
    def last_filler_ctas(self) -> int:
        return int(_lib().vx_last_filler_ctas(self.h))

    def timing(self, on: bool = True):
        _check(_lib().vx_timing_enable(self.h, 1 if on else 0))

    def integrator_time(self, reset: bool = True):
        """(summed device ms, launches) of integrator launches since the last reset."""
        ms, n = C.c_double(), C.c_int64()
        _check(_lib().vx_integrator_timing(self.h, C.byref(ms), C.byref(n), 1 if reset else 0))
        return float(ms.value), int(n.value)

    def decode_time(self, reset: bool = True):
        """(summed device ms, voxels decoded) of decode launches since the last reset."""
        ms, n = C.c_double(), C.c_int64()
        _check(_lib().vx_decode_timing(self.h, C.byref(ms), C.byref(n), 1 if reset else 0))
        return float(ms.value), int(n.value)

    def dmma_peak_tflops(self) -> float:
        t = C.c_double()
        _check(_lib().vx_dmma_peak(self.h, C.byref(t)))
        return float(t.value)

    def fp64_peak_tflops(self) -> float:
        t = C.c_double()
        _check(_lib().vx_fp64_peak(self.h, C.byref(t)))
        return float(t.value)

    def fastmath_check(self, n: int, seed: int = 1) -> tuple:
        """Mismatches (sqrt, rcp, fused sqrt+rcp) of the integrator's branch-free
        sqrt / reciprocal vs IEEE sqrt and division over n samples."""
        out = np.zeros(3, np.int64)
        _check(_lib().vx_fastmath_check(self.h, n, seed, out.ctypes.data))
        return int(out[0]), int(out[1]), int(out[2])

    def info(self) -> dict:
        sm, clk = C.c_int32(), C.c_int32()
        name = C.create_string_buffer(256)
        _check(_lib().vx_device_info(self.h, C.byref(sm), C.byref(clk), name, 256))
        return dict(sm_count=sm.value, clock_khz=clk.value, name=name.value.decode())


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------ decode etc.
def decode(genomes_params: np.ndarray, genomes_bmat: np.ndarray, arch: Arch, w: int, h: int, d: int,
           ctx: Optional[Context] = None):
    """decode (morphology.hpp:141-157) for P genomes -> (materials u8 P x cells, weights P x cells)."""
    ctx = ctx or default_context()
    params = np.ascontiguousarray(np.atleast_2d(genomes_params), np.float64)
    bmat = np.ascontiguousarray(np.atleast_2d(genomes_bmat), np.float64)
    P = params.shape[0]
    cells = w * h * d
    mat = np.zeros((P, cells), np.uint8)
    wt = np.zeros((P, cells))
    _check(_lib().vx_decode(ctx.h, C.byref(arch), P, _ptr(params), _ptr(bmat), w, h, d, _ptr(mat), _ptr(wt)), "decode")
    return mat, wt


def decode_refined(ctx: Optional[Context] = None) -> int:
    """Genomes of the context's last decode that the tensor-pipe path handed to
    the exact sequential path (a top-2 gap < 1e-8); -1 if that decode ran on
    the exact path only (VX_DECODE=exact, forward(), or weights too large)."""
    ctx = ctx or default_context()
    n = C.c_int64(0)
    _check(_lib().vx_decode_refined(ctx.h, C.byref(n)), "decode_refined")
    return int(n.value)


def gaussian_encode(v, bmat: np.ndarray, m: int) -> np.ndarray:
    """gaussian_encode(v, B, m) (genome.hpp:168-179) -> the 2m Fourier
    features of one point (host libm: bit-identical to the reference)."""
    vv = np.ascontiguousarray(v, np.float64).reshape(3)
    b = np.ascontiguousarray(bmat, np.float64).reshape(-1)
    if b.size != 3 * m:
        raise ShapeMismatch("gaussian_encode: encoding matrix size does not match m")
    out = np.zeros(2 * m)
    _check(_lib().vx_gaussian_encode(_ptr(vv), _ptr(b), int(m), _ptr(out)), "gaussian_encode")
    return out


def sample_genome(arch: Arch, seed: int, ctx: Optional[Context] = None):
    """sample_genome(spec, hidden, seed) (genome.hpp:146-166) -> (flat params,
    b_matrix); W bit-exact, B within ulps of glibc's normal()."""
    p, b = sample_genomes(arch, [seed], ctx)
    return p[0], b[0]


def sample_genomes(arch: Arch, seeds: Sequence[int], ctx: Optional[Context] = None):
    """sample_genome for many seeds in one launch -> (P x np params, P x 3m b_matrix)."""
    ctx = ctx or default_context()
    sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    P = len(sd)
    params = np.zeros((P, param_count(arch)))
    bmat = np.zeros((P, 3 * arch.m))
    _check(_lib().vx_sample_genomes(ctx.h, C.byref(arch), P, _ptr(sd), _ptr(params), _ptr(bmat)), "sample_genome")
    return params, bmat


def forward(params: np.ndarray, bmat: np.ndarray, arch: Arch, points: np.ndarray, ctx: Optional[Context] = None):
    """forward(genome, v) (genome.hpp:187-211), the pure spatial query, for
    one genome at many points (points: n x 3) or P genomes at n points each
    (params P x np, points P x n x 3) -> (probs [..., 5], weight [...])."""
    ctx = ctx or default_context()
    single = np.asarray(params).ndim == 1
    prm = np.ascontiguousarray(np.atleast_2d(params), np.float64)
    bm = np.ascontiguousarray(np.atleast_2d(bmat), np.float64)
    P = prm.shape[0]
    pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(P, -1, 3))
    n = pts.shape[1]
    probs = np.zeros((P, n, NMAT))
    wt = np.zeros((P, n))
    _check(_lib().vx_forward(ctx.h, C.byref(arch), P, _ptr(prm), _ptr(bm), n, _ptr(pts), _ptr(probs), _ptr(wt)),
           "forward")
    return (probs[0], wt[0]) if single else (probs, wt)


class Rng:
    """Rng (rng.hpp:15-56) over the library's host mt19937_64: next_u64,
    uniform01, normal (Box-Muller, glibc), index, text state interoperable
    with the reference's Rng::state / set_state."""

    def __init__(self, seed: int = 0):
        h = C.c_void_p()
        _check(_lib().vx_rng_create(int(seed), C.byref(h)), "Rng")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            _lib().vx_rng_free(self.h)
            self.h = None

    def next_u64(self) -> int:
        return int(_lib().vx_rng_next_u64(self.h))

    def uniform01(self) -> float:
        return float(_lib().vx_rng_uniform01(self.h))

    def normal(self) -> float:
        return float(_lib().vx_rng_normal(self.h))

    def index(self, n: int) -> int:
        if n <= 0:
            raise ValueError("Rng::index: n must be positive")
        return int(_lib().vx_rng_index(self.h, int(n)))

    def state(self) -> str:
        n = _lib().vx_rng_state(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        _lib().vx_rng_state(self.h, buf, int(n) + 1)
        return buf.value.decode()

    def set_state(self, s: str):
        _check(_lib().vx_rng_set_state(self.h, s.encode()), "Rng::set_state")

    def __eq__(self, other) -> bool:
        return isinstance(other, Rng) and self.state() == other.state()


def crossover(a_params: np.ndarray, b_params: np.ndarray, rng: Rng, a_bmat: Optional[np.ndarray] = None,
              b_bmat: Optional[np.ndarray] = None):
    """crossover(a, b, rng) (evolution.hpp:143-155): uniform per-parameter mix,
    the encoding matrix copied from a.  Returns the child's params (and its
    b_matrix when a_bmat is given).  Parents of different architecture raise
    ShapeMismatch."""
    a = np.ascontiguousarray(a_params, np.float64)
    b = np.ascontiguousarray(b_params, np.float64)
    if a.shape != b.shape or (a_bmat is not None and b_bmat is not None and np.shape(a_bmat) != np.shape(b_bmat)):
        raise ShapeMismatch("crossover: parents differ in architecture")
    child = np.empty_like(a)
    _check(_lib().vx_crossover(rng.h, a.size, _ptr(a), _ptr(b), _ptr(child)), "crossover")
    return child if a_bmat is None else (child, np.array(a_bmat, np.float64, copy=True))


def mutate(params: np.ndarray, rate: float, scale: float, rng: Rng) -> None:
    """mutate(g, rate, scale, rng) (evolution.hpp:160-165), in place."""
    if not (isinstance(params, np.ndarray) and params.dtype == np.float64 and params.flags.c_contiguous):
        raise ValueError("mutate: params must be a contiguous float64 array (mutated in place)")
    _check(_lib().vx_mutate(rng.h, params.size, _ptr(params), float(rate), float(scale)), "mutate")


def tournament_select(population: int, size: int, rng: Rng) -> int:
    """tournament_select(pop, size, rng) (evolution.hpp:169-173): index of the
    winner in the best-first sorted population of `population` individuals."""
    if population < 1:
        raise ValueError("tournament_select: empty population")
    return int(_lib().vx_tournament_select(rng.h, int(population), int(size)))


def largest_component(mats: np.ndarray, w: int, h: int, d: int, ctx: Optional[Context] = None) -> np.ndarray:
    """largest_component (morphology.hpp:162-208) for P grids."""
    ctx = ctx or default_context()
    mats = np.ascontiguousarray(np.atleast_2d(mats), np.uint8)
    out = np.zeros_like(mats)
    _check(_lib().vx_largest_component(ctx.h, mats.shape[0], w, h, d, _ptr(mats), _ptr(out)), "largest_component")
    return out


@dataclass
class SystemArrays:
    """Compact host view of a MassSpringSystem batch (morphology.hpp:110-135)."""
    mass_off: np.ndarray
    spring_off: np.ndarray
    pos: np.ndarray
    vel: np.ndarray
    mass: np.ndarray
    si: np.ndarray
    sj: np.ndarray
    k: np.ndarray
    rest0: np.ndarray
    zeta: np.ndarray
    has_act: np.ndarray
    sign: np.ndarray
    amp: np.ndarray
    phase: np.ndarray

    def robot(self, r: int) -> dict:
        m0, m1 = self.mass_off[r], self.mass_off[r + 1]
        s0, s1 = self.spring_off[r], self.spring_off[r + 1]
        out = {k: getattr(self, k)[m0:m1] for k in ("pos", "vel", "mass")}
        out.update({k: getattr(self, k)[s0:s1] for k in
                    ("si", "sj", "k", "rest0", "zeta", "has_act", "sign", "amp", "phase")})
        return out


class Batch:
    """Device-resident batch of mass-spring systems (vx_batch)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib().vx_batch_free(self.h)
                self.h = None
        except Exception:
            pass

    def __len__(self):
        return int(_lib().vx_batch_count(self.h))

    def offsets(self):
        n = len(self)
        mo = np.zeros(n + 1, np.int64)
        so = np.zeros(n + 1, np.int64)
        _check(_lib().vx_batch_offsets(self.h, _ptr(mo), _ptr(so)))
        return mo, so

    def download(self) -> SystemArrays:
        mo, so = self.offsets()
        M, S = int(mo[-1]), int(so[-1])
        a = SystemArrays(mass_off=mo, spring_off=so, pos=np.zeros((M, 3)), vel=np.zeros((M, 3)), mass=np.zeros(M),
                         si=np.zeros(S, np.int32), sj=np.zeros(S, np.int32), k=np.zeros(S), rest0=np.zeros(S),
                         zeta=np.zeros(S), has_act=np.zeros(S, np.uint8), sign=np.zeros(S), amp=np.zeros(S),
                         phase=np.zeros(S))
        _check(_lib().vx_batch_download(self.h, *[_ptr(getattr(a, f)) for f in
                                                  ("pos", "vel", "mass", "si", "sj", "k", "rest0", "zeta", "has_act",
                                                   "sign", "amp", "phase")]), "download")
        return a

    def workspace(self) -> dict:
        mo, so = self.offsets()
        M, S, n = int(mo[-1]), int(so[-1]), len(self)
        out = dict(damp_coef=np.zeros(S), amp_rest=np.zeros(S), sin_phase=np.zeros(S), cos_phase=np.zeros(S),
                   ground_damp=np.zeros(M), inc_off=np.zeros(M + n, np.int32), inc_spring=np.zeros(2 * S, np.int32),
                   inc_sign=np.zeros(2 * S))
        _check(_lib().vx_batch_workspace(self.h, *[_ptr(out[k]) for k in
                                                   ("damp_coef", "amp_rest", "sin_phase", "cos_phase", "ground_damp",
                                                    "inc_off", "inc_spring", "inc_sign")]), "workspace")
        return out

    def set_state(self, pos: np.ndarray, vel: Optional[np.ndarray] = None):
        pos = np.ascontiguousarray(pos, np.float64)
        vel = None if vel is None else np.ascontiguousarray(vel, np.float64)
        _check(_lib().vx_batch_set_state(self.h, _ptr(pos), _ptr(vel)))

    def override_phase(self, sin_phase: np.ndarray, cos_phase: np.ndarray):
        s = np.ascontiguousarray(sin_phase, np.float64)
        c = np.ascontiguousarray(cos_phase, np.float64)
        _check(_lib().vx_batch_override_phase(self.h, _ptr(s), _ptr(c)))

    def step(self, sim: SimConfig, k0: int = 0, n_steps: int = 1):
        """step() (physics.hpp:191-264) n_steps times from t = k0*dt; mutates the batch."""
        out = (TrajectorySummary * max(1, len(self)))()
        _check(_lib().vx_batch_step(self.ctx.h, self.h, C.byref(sim), k0, n_steps, out), "step")
        return list(out)[:len(self)]

    def step_at(self, sim: SimConfig, t: float):
        """step(sys, t, cfg, ws) (physics.hpp:191-264) once at an arbitrary time t; mutates the batch."""
        out = (TrajectorySummary * max(1, len(self)))()
        _check(_lib().vx_batch_step_at(self.ctx.h, self.h, C.byref(sim), float(t), out), "step_at")
        return list(out)[:len(self)]

    def simulate(self, sim: SimConfig):
        """simulate() (physics.hpp:287-311) for every robot (batch unchanged)."""
        out = (TrajectorySummary * max(1, len(self)))()
        _check(_lib().vx_batch_simulate(self.ctx.h, self.h, C.byref(sim), out), "simulate")
        return list(out)[:len(self)]

    def simulate_dump(self, sim: SimConfig, stride: int):
        """simulate(sys, cfg, &dump, stride) (physics.hpp:280-311) for every
        robot: returns (summaries, dumps) with dumps[r] an (rows, 4) array of
        TrajectorySample (t, com x, y, z).  The batch is unchanged."""
        n = len(self)
        n_steps = int(math.floor(sim.duration / sim.dt + 0.5)) if sim.dt > 0 else 0  # llround
        cap = (-(-n_steps // stride) if stride > 0 else 0) + 1
        rows = np.zeros((max(1, n), cap, 4))
        counts = np.zeros(max(1, n), np.int64)
        out = (TrajectorySummary * max(1, n))()
        _check(_lib().vx_batch_simulate_dump(self.ctx.h, self.h, C.byref(sim), int(stride), cap, _ptr(rows),
                                             _ptr(counts), out), "simulate_dump")
        return list(out)[:n], [rows[r, :min(int(counts[r]), cap)].copy() for r in range(n)]

    def simulate_dev(self, sim: SimConfig, d_summaries: int):
        _check(_lib().vx_batch_simulate_dev(self.ctx.h, self.h, C.byref(sim), d_summaries), "simulate_dev")


def build_mass_spring(mats: np.ndarray, weights: np.ndarray, w: int, h: int, d: int,
                      table: Optional[MaterialTable] = None, plane: Optional[GroundPlane] = None,
                      ctx: Optional[Context] = None) -> Batch:
    """build_mass_spring (morphology.hpp:217-299) for P body grids."""
    ctx = ctx or default_context()
    mats = np.ascontiguousarray(np.atleast_2d(mats), np.uint8)
    weights = np.ascontiguousarray(np.atleast_2d(weights), np.float64)
    table = table or MaterialTable()
    plane = plane or GroundPlane()
    hb = C.c_void_p()
    _check(_lib().vx_batch_build(ctx.h, mats.shape[0], w, h, d, _ptr(mats), _ptr(weights), C.byref(table),
                                 C.byref(plane), C.byref(hb)), "build_mass_spring")
    return Batch(hb, ctx)


def upload_systems(systems: Sequence, plane: Optional[GroundPlane] = None, ctx: Optional[Context] = None) -> Batch:
    """Upload host-assembled systems (objects with pos, vel, mass, si, sj, k,
    rest0, zeta, has_act, sign, amp, phase — e.g. oracle.System)."""
    ctx = ctx or default_context()
    plane = plane or GroundPlane()
    n = len(systems)
    mo = np.zeros(n + 1, np.int64)
    so = np.zeros(n + 1, np.int64)
    for r, s in enumerate(systems):
        mo[r + 1] = mo[r] + len(s.mass)
        so[r + 1] = so[r] + len(s.k)

    def cat(f, dt, shape=None):
        parts = [np.asarray(getattr(s, f), dt).reshape(-1) for s in systems]
        return np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(0, dt))

    arrs = [cat("pos", np.float64), cat("vel", np.float64), cat("mass", np.float64), cat("si", np.int32),
            cat("sj", np.int32), cat("k", np.float64), cat("rest0", np.float64), cat("zeta", np.float64),
            cat("has_act", np.uint8), cat("sign", np.float64), cat("amp", np.float64), cat("phase", np.float64)]
    hb = C.c_void_p()
    _check(_lib().vx_batch_upload(ctx.h, n, _ptr(mo), _ptr(so), *[_ptr(a) for a in arrs], C.byref(plane),
                                  C.byref(hb)), "upload")
    return Batch(hb, ctx)


def evaluate_fitness(mats: np.ndarray, weights: np.ndarray, w: int, h: int, d: int,
                     table: Optional[MaterialTable] = None, plane: Optional[GroundPlane] = None,
                     sim: Optional[SimConfig] = None, ctx: Optional[Context] = None, with_summaries: bool = False):
    """evaluate_fitness (evolution.hpp:110-119) for P raw grids."""
    ctx = ctx or default_context()
    mats = np.ascontiguousarray(np.atleast_2d(mats), np.uint8)
    weights = np.ascontiguousarray(np.atleast_2d(weights), np.float64)
    P = mats.shape[0]
    table = table or MaterialTable()
    plane = plane or GroundPlane()
    sim = sim or SimConfig()
    fit = np.zeros(P)
    summ = (TrajectorySummary * max(1, P))() if with_summaries else None
    _check(_lib().vx_evaluate(ctx.h, P, w, h, d, _ptr(mats), _ptr(weights), C.byref(table), C.byref(plane),
                              C.byref(sim), _ptr(fit), summ), "evaluate_fitness")
    return (fit, list(summ)[:P]) if with_summaries else fit


def population_diversity(mats: np.ndarray, ctx: Optional[Context] = None) -> float:
    """population_diversity (evolution.hpp:89-105) over P raw grids."""
    ctx = ctx or default_context()
    mats = np.ascontiguousarray(np.atleast_2d(mats), np.uint8)
    out = C.c_double()
    _check(_lib().vx_population_diversity(ctx.h, mats.shape[0], mats.shape[1], _ptr(mats), C.byref(out)))
    return float(out.value)


def run_bench(jobs: int = 16, steps: int = 2000, grid: int = 4, dt: float = 1e-5,
              ctx: Optional[Context] = None) -> dict:
    """run_bench (bench.hpp:50-86) on device."""
    ctx = ctx or default_context()
    out = np.zeros(6)
    _check(_lib().vx_run_bench(ctx.h, jobs, steps, grid, dt, _ptr(out)), "run_bench")
    return dict(springs_per_robot=int(out[0]), spring_updates=int(out[1]), expected_updates=int(out[2]),
                seconds=float(out[3]), updates_per_second=float(out[4]), diverged=bool(out[5]))


# ----------------------------------------------------------------- evolution
AdvisorFn = Callable[[list, HyperParams], Optional[HyperParams]]
ADVISOR_WINDOW = 3  # kAdvisorWindow (evolution.hpp:195)


class EvolutionState:
    """init_evolution / evolve_generation (evolution.hpp:177-293), device-resident."""

    def __init__(self, config: EvolutionConfig, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.config = config
        h = C.c_void_p()
        _check(_lib().vx_evo_create(self.ctx.h, C.byref(config), C.byref(h)), "init_evolution")
        self.h = h
        self.history: list = []
        self.np = param_count(config.arch)
        self.cells = config.grid_w * config.grid_h * config.grid_d

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib().vx_evo_free(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def generation(self) -> int:
        return int(_lib().vx_evo_generation_index(self.h))

    @property
    def params(self) -> HyperParams:
        p = HyperParams()
        _check(_lib().vx_evo_get_params(self.h, C.byref(p)))
        return p

    @params.setter
    def params(self, p: HyperParams):
        _check(_lib().vx_evo_set_params(self.h, C.byref(p)))

    def best(self):
        bf = C.c_double()
        bp = np.zeros(self.np)
        has = _lib().vx_evo_best(self.h, C.byref(bf), _ptr(bp))
        return float(bf.value), (bp if has else None)

    def _best_bmat(self):
        bf = C.c_double()
        bp = np.zeros(self.np)
        bb = np.zeros(3 * self.config.arch.m)
        has = _lib().vx_evo_best_genome(self.h, C.byref(bf), _ptr(bp), _ptr(bb))
        return bb if has else None

    def set_progress(self, generation: int, best_fitness: float, best=None):
        """Resume support: generation counter and best_fitness / best_genome
        (``best`` = (params, bmat) or None)."""
        if best is None:
            _check(_lib().vx_evo_set_progress(self.h, int(generation), float(best_fitness), None, None),
                   "set_progress")
        else:
            bp = np.ascontiguousarray(best[0], np.float64)
            bb = np.ascontiguousarray(best[1], np.float64)
            if bp.size != self.np or bb.size != 3 * self.config.arch.m:
                raise ValueError("best genome shape does not match the architecture")
            _check(_lib().vx_evo_set_progress(self.h, int(generation), float(best_fitness), _ptr(bp), _ptr(bb)),
                   "set_progress")

    def rng_state(self) -> str:
        n = _lib().vx_evo_rng_state(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        _lib().vx_evo_rng_state(self.h, buf, int(n) + 1)
        return buf.value.decode()

    def set_rng_state(self, s: str):
        _check(_lib().vx_evo_set_rng_state(self.h, s.encode()), "set_rng_state")

    def population(self) -> dict:
        P, cells = self.config.population, self.cells
        out = dict(params=np.zeros((P, self.np)), bmat=np.zeros((P, 3 * self.config.arch.m)), fitness=np.zeros(P),
                   evaluated=np.zeros(P, np.uint8), grids=np.zeros((P, cells), np.uint8), grid_w=np.zeros((P, cells)))
        _check(_lib().vx_evo_get_population(self.h, *[_ptr(out[k]) for k in
                                                      ("params", "bmat", "fitness", "evaluated", "grids", "grid_w")]))
        return out

    def get_population_into(self, params, bmat, fitness=None, evaluated=None):
        """Copy the population into caller arrays (e.g. pinned host memory):
        params (P, np) f64, bmat (P, 3m) f64, fitness (P,) f64, evaluated (P,) u8."""
        P = self.config.population
        checks = [(params, (P, self.np), np.float64), (bmat, (P, 3 * self.config.arch.m), np.float64),
                  (fitness, (P,), np.float64), (evaluated, (P,), np.uint8)]
        for a, shape, dt in checks:
            if a is not None and (a.shape != shape or a.dtype != dt or not a.flags.c_contiguous):
                raise ValueError(f"get_population_into: expected a C-contiguous {dt.__name__} array of shape {shape}")
        _check(_lib().vx_evo_get_population(self.h, _ptr(params), _ptr(bmat), _ptr(fitness), _ptr(evaluated), None,
                                            None), "get_population")

    def set_population(self, params, bmat, fitness=None, evaluated=None, grids=None, grid_w=None):
        c = np.ascontiguousarray
        arrs = [c(params, np.float64), c(bmat, np.float64), None if fitness is None else c(fitness, np.float64),
                None if evaluated is None else c(evaluated, np.uint8), None if grids is None else c(grids, np.uint8),
                None if grid_w is None else c(grid_w, np.float64)]
        _check(_lib().vx_evo_set_population(self.h, *[_ptr(a) for a in arrs]), "set_population")

    def _advise(self, advisor: Optional[AdvisorFn]):
        # evolution.hpp:221-227: consult with the trailing window once enough history exists
        if advisor is not None and len(self.history) >= ADVISOR_WINDOW:
            adjusted = advisor(self.history[-ADVISOR_WINDOW:], self.params)
            if adjusted is not None:
                self.params = adjusted  # clamped by the library

    def evolve_generation(self, advisor: Optional[AdvisorFn] = None) -> GenerationReport:
        self._advise(advisor)
        rep = GenerationReport()
        _check(_lib().vx_evo_generation(self.h, C.byref(rep)), "evolve_generation")
        self.history.append(rep)
        return rep

    # sharded form: begin -> all-reduce(exchange) -> finish
    def begin(self, rank: int, world: int, advisor: Optional[AdvisorFn] = None):
        self._advise(advisor)
        _check(_lib().vx_evo_begin(self.h, rank, world), "evo_begin")

    def exchange_buffer(self):
        p = C.c_void_p()
        n = C.c_int64()
        _check(_lib().vx_evo_exchange_buffer(self.h, C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)

    def set_exchange_buffer(self, d_ptr: int):
        """Use a caller-owned device buffer of exchange_buffer()[1] doubles (e.g. a torch tensor
        that torch.distributed all-reduces) as the exchange buffer."""
        _check(_lib().vx_evo_set_exchange_buffer(self.h, d_ptr))

    def load_population_dev(self, d_params: int, d_bmat: int):
        """Generation-0 reset from device arrays (init_evolution state)."""
        _check(_lib().vx_evo_load_population_dev(self.h, d_params, d_bmat), "load_population_dev")

    def finish(self) -> GenerationReport:
        rep = GenerationReport()
        _check(_lib().vx_evo_finish(self.h, C.byref(rep)), "evo_finish")
        self.history.append(rep)
        return rep

    def set_comm(self, comm: Optional["Communicator"]):
        """Shard every evolve_generation over the communicator's ranks (NCCL
        all-reduce of the exchange buffer inside the library)."""
        self._comm = comm
        _check(_lib().vx_evo_set_comm(self.h, comm.h if comm is not None else None), "set_comm")

    def set_exchange(self, rank: int, world: int, fn: Optional[Callable[[int, int], None]]):
        """Shard over any transport: fn(d_buf_ptr, n_doubles) must leave the
        element-wise sum over all ranks in the device buffer."""
        if fn is None:
            self._xfn = None
            _check(_lib().vx_evo_set_exchange(self.h, 0, 1, None, None), "set_exchange")
            return

        def tramp(d_buf, n, _user):
            try:
                fn(int(d_buf or 0), int(n))
                return VX_OK
            except Exception:  # reported as a CUDA-side failure of the exchange
                return VX_ECUDA
        self._xfn = _EXCHANGE_FN(tramp)
        _check(_lib().vx_evo_set_exchange(self.h, rank, world, self._xfn, None), "set_exchange")


_EXCHANGE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_void_p)


def _nccl_lib():
    """The library resolves NCCL at first use and prefers one already in the
    process: make that PyTorch's (importing torch after the system NCCL was
    loaded would bind torch to the older copy)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    return _lib()


class Communicator:
    """NCCL communicator of one rank (vx_comm_create): population sharding
    across GPUs, one process per GPU."""

    @staticmethod
    def available() -> bool:
        return _nccl_lib().vx_comm_available() == VX_OK

    @staticmethod
    def unique_id() -> bytes:
        _nccl_lib()
        buf = (C.c_uint8 * 128)()
        _check(_lib().vx_comm_unique_id(buf), "comm_unique_id")
        return bytes(buf)

    def __init__(self, ctx: "Context", world: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.ctx = ctx
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(_lib().vx_comm_create(ctx.h, world, rank, buf, C.byref(h)), "comm_create")
        self.h = h
        self.rank, self.world = rank, world

    def allreduce_sum_dev(self, d_ptr: int, n: int):
        _check(_lib().vx_comm_allreduce_sum_dev(self.h, d_ptr, n), "comm_allreduce")

    def close(self):
        if getattr(self, "h", None):
            _lib().vx_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_indices(todo: Sequence[int], rank: int, world: int) -> list:
    """The children a rank evaluates in vx_evo_begin(rank, world): a strided
    split of the generation's todo list (every index exactly once)."""
    return [int(t) for t in list(todo)[rank::world]]


def init_evolution(config: EvolutionConfig, ctx: Optional[Context] = None) -> EvolutionState:
    return EvolutionState(config, ctx)


def evolve_generation(state: EvolutionState, advisor: Optional[AdvisorFn] = None) -> GenerationReport:
    return state.evolve_generation(advisor)


def report_dict(r: GenerationReport) -> dict:
    return dict(generation=r.generation, evaluations=r.evaluations, best=r.best, mean=r.mean, stddev=r.stddev,
                diversity=r.diversity, wall_time=r.wall_time, spring_updates=int(r.spring_updates),
                params=r.params.as_array())


# config files and checkpoints (config.hpp / serialize.hpp formats)
from .serialize import (CheckpointError, ConfigError, RunConfig, curves_csv, load_genome, load_run,  # noqa: E402
                        load_run_config, run_config_from_json, save_genome, save_run, write_curves_csv)
from .runner import ScriptedAdvisor, resume_run, run_config_to_json, run_loop, start_run  # noqa: E402
