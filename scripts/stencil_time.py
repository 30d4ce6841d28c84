"""Device time of apply_stencil on config 2 (cube-kuhn L8), CUDA events, for
kernel development (env BT_STENCIL_PARTS / BT_PRISM_MODE select parts).
   python scripts/stencil_time.py [reps] [level]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_01792_b200 as bt  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
l = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = bt.Grid(bt.cube_kuhn_text(), l, l, device=0)
x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
bt.random_fill(x, l, 0)
t = bt.compute_stencil(bt.FormId.diffusion(), g, l)
for _ in range(10):
    bt.apply_stencil(t, x, y, l)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    bt.apply_stencil(t, x, y, l)
b.record()
torch.cuda.synchronize()
print(f"parts={os.environ.get('BT_STENCIL_PARTS', '15')} mode={os.environ.get('BT_PRISM_MODE', '0')} "
      f"us/apply={a.elapsed_time(b) / reps * 1e3:.1f}")
