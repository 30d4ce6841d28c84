"""Device time of the N1E1 apply on config 4 (384 perturbed tets, L7).
   python scripts/n1e1_time.py [reps] [level]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_01792_b200 as bt  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
l = int(sys.argv[2]) if len(sys.argv) > 2 else 7
g = bt.Grid(bt.cubes_mesh_text(4, 0.1, 0), l, l, device=0)
op = bt.N1E1Operator(g, l)
x, y = bt.allocate(bt.edge_space(), g, l, l), bt.allocate(bt.edge_space(), g, l, l)
bt.random_fill(x, l, 0)
for _ in range(3):
    bt.apply_n1e1(op, x, y, l)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    bt.apply_n1e1(op, x, y, l)
b.record()
torch.cuda.synchronize()
print(f"N1E1 L{l}: ms/apply={a.elapsed_time(b) / reps:.3f}")
