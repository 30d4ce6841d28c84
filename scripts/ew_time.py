"""Device time of apply_elementwise(div k grad) on config 3 (384 perturbed
tets, L6), CUDA events, for kernel development.
   python scripts/ew_time.py [reps] [level] [ncubes]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_01792_b200 as bt  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
l = int(sys.argv[2]) if len(sys.argv) > 2 else 6
nc = int(sys.argv[3]) if len(sys.argv) > 3 else 4
g = bt.Grid(bt.cubes_mesh_text(nc, 0.1, 0), l, l, device=0)
x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
bt.random_fill(x, l, 0)
f = bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.0, 0.5, 2 * np.pi))
for _ in range(3):
    bt.apply_elementwise(f, x, y, l)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    bt.apply_elementwise(f, x, y, l)
b.record()
torch.cuda.synchronize()
print(f"L{l} {nc}^3 cubes: us/apply={a.elapsed_time(b) / reps * 1e3:.1f}")
