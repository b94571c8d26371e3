"""A/B of the decode kernels at the config-3 shape (P genomes -> 10^3 grids):
the DMMA tensor-pipe kernel (default) vs the exact sequential-order CUDA-core
kernel (VX_DECODE=exact).  Device buffers, CUDA events on the context stream;
prints ms per decode and the MLP's achieved FP64 TFLOP/s (2 x 8,576 MAC per
voxel for the default network) and checks both paths agree.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00698_b200 as vx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=4096)
    ap.add_argument("--grid", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    ctx = vx.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    arch = vx.Arch.make()
    seeds = [int(x) for x in np.random.default_rng(1).integers(0, 2 ** 62, args.P)]
    params, bmat = vx.sample_genomes(arch, seeds, ctx)
    g = args.grid
    cells = g ** 3
    dp = torch.from_numpy(params).cuda()
    db = torch.from_numpy(bmat).cuda()
    lib = vx._lib()
    mac = 2 * 32 * 64 + 64 * 64 + 64 * 6
    out = {}
    for mode in ("mma", "exact"):
        if mode == "exact":
            os.environ["VX_DECODE"] = "exact"
        else:
            os.environ.pop("VX_DECODE", None)
        dm = torch.zeros(args.P * cells, dtype=torch.uint8, device="cuda")
        dw = torch.zeros(args.P * cells, dtype=torch.float64, device="cuda")
        times = []
        for r in range(args.reps + 1):
            with torch.cuda.stream(s):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                st = lib.vx_decode_dev(ctx.h, C.byref(arch), args.P, C.c_void_p(dp.data_ptr()),
                                       C.c_void_p(db.data_ptr()), g, g, g, C.c_void_p(dm.data_ptr()),
                                       C.c_void_p(dw.data_ptr()), None)
                e1.record(s)
            assert st == 0, st
            s.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        out[mode] = (dm.cpu().numpy(), dw.cpu().numpy())
        tf = 2.0 * mac * cells * args.P / (ms * 1e-3) / 1e12
        print(f"{mode:5s}: P={args.P} {g}^3  {ms:8.3f} ms/decode  MLP {tf:6.2f} TFLOP/s  "
              f"refined={vx.decode_refined(ctx)}")
    os.environ.pop("VX_DECODE", None)
    same = np.array_equal(out["mma"][0], out["exact"][0])
    rel = np.max(np.abs(out["mma"][1] - out["exact"][1]) / np.abs(out["exact"][1]))
    print(f"materials identical: {same}; weights max rel diff {rel:.3e}")


if __name__ == "__main__":
    main()
