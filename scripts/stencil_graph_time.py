"""Device time of apply_stencil on config 2 replayed from a CUDA graph of 10 applies (no CPU launch cost), next to
the eager loop. python scripts/stencil_graph_time.py [level]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_01792_b200 as bt  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = bt.Grid(bt.cube_kuhn_text(), l, l, device=0)
x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
bt.random_fill(x, l, 0)
t = bt.compute_stencil(bt.FormId.diffusion(), g, l)
for _ in range(10):
    bt.apply_stencil(t, x, y, l)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(500):
    bt.apply_stencil(t, x, y, l)
b.record()
torch.cuda.synchronize()
eager = a.elapsed_time(b) / 500 * 1e3
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(gr, stream=s):
        for _ in range(10):
            bt.apply_stencil(t, x, y, l)
torch.cuda.synchronize()
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
a.record()
for _ in range(50):
    gr.replay()
b.record()
torch.cuda.synchronize()
print(f"level {l} parts={os.environ.get('BT_STENCIL_PARTS', '15')}: eager {eager:.1f} us/apply, graph "
      f"{a.elapsed_time(b) / 500 * 1e3:.1f} us/apply")
