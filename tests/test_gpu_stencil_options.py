"""The fast stencil march's opt-in schedules and the warp-marched strided faces give bitwise the default apply.

The knobs are read once per process (BT_STENCIL_SCHED: 0 round-robin 32-row marches (default), 1 balanced per-warp
lists, 2 dynamic queue; BT_STENCIL_MARCH; BT_STENCIL_FACEMARCH), so each case runs in its own interpreter and
prints a digest of y for cube-kuhn at level 8 (config 2), with and without Dirichlet identity rows.
"""
import hashlib
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import hashlib, torch, paper_2308_01792_b200 as bt
l = 8
g = bt.Grid(bt.cube_kuhn_text(), l, l, device=0)
x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
bt.random_fill(x, l, 0)
t = bt.compute_stencil(bt.FormId.diffusion(), g, l)
out = []
for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
    y.values[l].zero_()
    bt.apply_stencil(t, x, y, l, bc)
    bt.apply_stencil(t, x, y, l, bc)  # a second launch: the dynamic queue has reset itself
    torch.cuda.synchronize()
    out.append(hashlib.sha256(y.values[l].cpu().numpy().tobytes()).hexdigest())
print("DIGEST", *out)
'''


def _digest(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("DIGEST")][-1]
    return line.split()[1:]


@pytest.mark.gpu
def test_schedules_and_face_march_bitwise_default():
    ref = _digest({"BT_STENCIL_SCHED": "0"})
    assert len(ref) == 2 and ref[0] != ref[1]
    for env in ({"BT_STENCIL_SCHED": "1"}, {"BT_STENCIL_SCHED": "2"},
                {"BT_STENCIL_SCHED": "2", "BT_STENCIL_MARCH": "16"}, {"BT_STENCIL_FACEMARCH": "1"}):
        assert _digest(env) == ref, env
