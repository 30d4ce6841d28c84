"""Per-rank device time of the partitioned (fused) stencil apply against the
one-GPU apply, on one GPU: rank r of R over cube-kuhn L8 (6 cells) or an
R x 1 x 1 box of unit cubes (6 cells per rank), with an allreduce hook that
does nothing (it measures the rank's own work: interior, local boundary,
exchange partials and combine; the collective itself is what NVLink adds).
   python scripts/partition_time.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_01792_b200 as bt  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L = 8


def timed(text, rank, nranks):
    g = bt.Grid(text, L, L, device=0)
    if nranks > 1:
        g.set_partition(rank, nranks, allreduce=lambda t: None)
    x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, L, 0) if nranks == 1 else x.values[L].uniform_(-1, 1)
    t = bt.compute_stencil(bt.FormId.diffusion(), g, L)
    for _ in range(10):
        bt.apply_stencil(t, x, y, L)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        bt.apply_stencil(t, x, y, L)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3, x.values[L].numel()


one, s1 = timed(bt.cube_kuhn_text(), 0, 1)
print(f"1 GPU, 6 cells: {one:.1f} us ({s1} slots)")
for R in (2, 3):
    for r in range(R):
        us, s = timed(bt.cube_kuhn_text(), r, R)
        print(f"cube-kuhn rank {r}/{R}: {us:.1f} us for {s} slots; ideal {one * s / s1:.1f} us")
for R in (2, 4, 8):
    us, s = timed(bt.box_mesh_text(R, 1, 1), R // 2, R)
    print(f"box {R}x1x1 rank {R // 2}/{R} (6 cells): {us:.1f} us for {s} slots (1 GPU, 6 cells: {one:.1f} us)")
