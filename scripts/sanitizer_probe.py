import numpy as np, os, sys
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
import paper_2405_00698_b200 as vx
ctx = vx.Context(0)
arch = vx.Arch.make()
p, b = vx.sample_genomes(arch, [1, 2, 3, 4], ctx)
m, w = vx.decode(p, b, arch, 6, 6, 6, ctx)
print("decode ok", vx.decode_refined(ctx))
g = np.random.default_rng(0).integers(0, 5, (70, 200)).astype(np.uint8)
print("div", vx.population_diversity(g, ctx))
