"""Regenerate tests/golden/*.npz from the REFERENCE itself.

Runs the unmodified reference headers compiled by oracle/Makefile
(oracle/_ref/libvoxevo_ref.so) in this container.  The committed fixtures let
the CPU suite and the GPU box (where /root/reference is absent) pin the oracle
and the CUDA path without the reference tree.

    python tests/golden/make_golden.py

Host facts (glibc version, libm ifunc variant) are recorded in meta.json:
values that pass through glibc exp/log/sin/cos/tanh are only bit-stable on the
same libm variant (SURVEY.md summary item 5).
"""
import json
import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def sys_dict(s, prefix):
    return {f"{prefix}{k}": getattr(s, k) for k in
            ("pos", "vel", "mass", "si", "sj", "k", "rest0", "zeta", "has_act", "sign", "amp", "phase")}


def main():
    R = oracle.reference()
    out = {}
    # ---- rng KATs (rng.hpp)
    out["kat_5489_10000"] = R.rng_draws(5489, 10000)[-1:]
    out["kat_42_first"] = R.rng_draws(42, 8)
    out["rng7_uniform"] = R.rng_uniform(7, 64)
    out["rng7_normal"] = R.rng_normal(7, 64)
    out["rng9_index7"] = R.rng_index(9, 64, 7)
    state = R.rng_state(99, 17)
    out["rng99_state17"] = np.frombuffer(state.encode(), np.uint8)
    out["rng99_after17"] = R.rng_draws_from_state(state, 50)

    # ---- config 1: sample_genome(seed 42) -> decode 4^3 -> component -> build -> 1000 steps
    params, bmat = R.sample_genome(32, [64, 64], 42)
    mat, wt = R.decode(32, [64, 64], params, bmat, 4, 4, 4)
    body = R.largest_component(mat, 4, 4, 4)
    s = R.build(body, wt, 4, 4, 4)
    out["c1_params"] = params
    out["c1_bmat"] = bmat
    out["c1_mat"] = mat
    out["c1_wt"] = wt
    out["c1_body"] = body
    out.update(sys_dict(s, "c1_sys_"))
    ws = R.workspace(s)
    for k, v in ws.items():
        out["c1_ws_" + k] = v
    sim = oracle.sim6(duration=1000 * 1e-5)
    summ = R.simulate(s, sim)
    out["c1_summary"] = np.concatenate([summ["com_start"], summ["com_end"],
                                        [summ["horizontal_displacement"], summ["max_speed"], float(summ["diverged"])]])
    s100, ok, called, upd, msq = R.step(s, sim, 0, 100)
    out["c1_step100_pos"] = s100.pos
    out["c1_step100_vel"] = s100.vel
    out["c1_step100_meta"] = np.array([ok, called, upd, msq])

    # ---- bench_robot(4) (bench.hpp:35-44) and its system
    bm, bw = R.bench_robot(4)
    bs = R.build(bm, bw, 4, 4, 4)
    out["b4_mat"] = bm
    out.update(sys_dict(bs, "b4_sys_"))
    res = np.zeros(6)
    R._run_bench(16, 2000, 1, 4, 1e-5, res.ctypes.data)
    out["b4_bench_counts"] = res[[0, 1, 2, 5]]  # springs/robot, updates, expected, diverged

    # ---- unit-test KATs (test_morphology.cpp, test_evolution.cpp)
    out["elite_table"] = np.array([[0.3, 30, R.elite_count(0.3, 30)], [0.05, 12, R.elite_count(0.05, 12)],
                                   [0.31, 30, R.elite_count(0.31, 30)], [0.9, 2, R.elite_count(0.9, 2)],
                                   [0.05, 100, R.elite_count(0.05, 100)]])

    # ---- config-2-shaped population (P=8 of 6^3, seed 42): decode + build topology
    ev = R.evo(population=8, generations=0, grid=(6, 6, 6), seed=42)
    pop = ev.population()
    out["c2_params"] = pop["params"]
    out["c2_bmat"] = pop["bmat"]
    mats = []
    wts = []
    for a in range(8):
        m_, w_ = R.decode(32, [64, 64], pop["params"][a], pop["bmat"][a], 6, 6, 6)
        mats.append(m_)
        wts.append(w_)
    out["c2_mat"] = np.stack(mats)
    out["c2_wt"] = np.stack(wts)
    nms, nss = [], []
    for a in range(8):
        b_ = R.largest_component(mats[a], 6, 6, 6)
        sy = R.build(b_, wts[a], 6, 6, 6)
        nms.append(0 if sy is None else sy.nm)
        nss.append(0 if sy is None else sy.ns)
    out["c2_nm"] = np.array(nms)
    out["c2_ns"] = np.array(nss)
    out["c2_diversity"] = np.array([R.population_diversity(out["c2_mat"])])

    # ---- desk GA (acceptance_main.cpp:193-211 shape, seed 1), reports per generation
    ev = R.evo(population=12, generations=20, grid=(3, 3, 3), seed=1, sim=oracle.sim6(dt=1e-4, duration=0.5))
    reps = [ev.generation() for _ in range(21)]
    out["desk1_best"] = np.array([r["best"] for r in reps])
    out["desk1_mean"] = np.array([r["mean"] for r in reps])
    out["desk1_div"] = np.array([r["diversity"] for r in reps])
    out["desk1_evals"] = np.array([r["evaluations"] for r in reps])
    out["desk1_rng_state"] = np.frombuffer(ev.rng_state().encode(), np.uint8)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    meta = dict(
        generator="tests/golden/make_golden.py",
        reference="/root/reference/proj/include/voxevo (unmodified), via oracle/ref_shim.cpp",
        flags="g++ -std=c++20 -O2 -ffp-contract=off (no -march)",
        glibc=platform.libc_ver()[1],
        libm_variant=("default ifunc (" + ("FMA/AVX2 host" if "fma" in open("/proc/cpuinfo").read() else "SSE2 host")
                      + "), GLIBC_TUNABLES=" + os.environ.get("GLIBC_TUNABLES", "<unset>")),
        note="libm-dependent values (weights, normals, trajectories, fitness) are bit-stable only on the same "
             "glibc + ifunc variant; integer/topology values are host-independent.",
    )
    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")


if __name__ == "__main__":
    main()
