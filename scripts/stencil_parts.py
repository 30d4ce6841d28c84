"""Time the parts of the config-2 stencil apply (profiling aid): run once per
BT_STENCIL_PARTS mask in a fresh process; prints mean us per apply_stencil (fused path)."""
import json
import os
import subprocess
import sys

CODE = r'''
import torch, json, paper_2308_01792_b200 as bt
from paper_2308_01792_b200 import _lib
L = 8
g = bt.Grid(bt.cube_kuhn_text(), L, L)
t = bt.compute_stencil(bt.FormId.diffusion(), g, L)
x = bt.allocate(bt.p1_space(), g); y = bt.allocate(bt.p1_space(), g)
bt.random_fill(x, L, 0)
xp, yp = bt.api._ptr(x.values[L]), bt.api._ptr(y.values[L])
for _ in range(20): _lib.lib.bt_apply_stencil(t.handle, xp, yp, 0, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 2000
e0.record()
for _ in range(K): _lib.lib.bt_apply_stencil(t.handle, xp, yp, 0, None)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"us": e0.elapsed_time(e1) / K * 1e3}))
'''

if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for mask, name in [(1, "interior"), (8, "boundary"), (9, "both")]:
        env = dict(os.environ, BT_STENCIL_PARTS=str(mask))
        r = subprocess.run([sys.executable, "-c", CODE], cwd=root, env=env, capture_output=True, text=True)
        try:
            us = json.loads(r.stdout.strip().splitlines()[-1])["us"]
            print(f"{name:14s} {us:8.2f} us")
        except Exception:
            print(name, "failed", r.stderr[-500:])
