"""Device time of the bit-exact population_diversity (csrc/diversity.cu) at
the bench shapes: random 10^3 grids, P = 4096 (config 3), 32768 (config 3 on
8 GPUs), 65536 (config 4).  CUDA events on the context stream."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_00698_b200 as vx  # noqa: E402


def main():
    ctx = vx.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    lib = vx._lib()
    cells = 1000
    for P in [int(x) for x in (sys.argv[1:] or ["4096", "32768", "65536"])]:
        g = torch.randint(0, 5, (P, cells), dtype=torch.uint8, device="cuda")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        times = []
        for rep in range(3):
            with torch.cuda.stream(s):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                st = lib.vx_population_diversity_dev(ctx.h, P, cells, C.c_void_p(g.data_ptr()),
                                                     C.c_void_p(out.data_ptr()))
                e1.record(s)
            assert st == 0
            s.synchronize()
            times.append(e0.elapsed_time(e1))
        print(f"P={P} cells={cells} pairs={P * (P - 1) // 2}: {min(times):.3f} ms (diversity {out.item():.17g})")


if __name__ == "__main__":
    main()
