"""CUDA-graph capture of the public applies (bench_configs.py times config 1
from a graph): replays are bitwise the eager results, for the single-launch
small path, the two-stream fused path, the elementwise path and N1E1."""
import math

import pytest
import torch

import paper_2308_01792_b200 as bt

pytestmark = pytest.mark.gpu


def replay_equals_eager(run, out):
    run()
    torch.cuda.synchronize()
    eager = out.clone()
    out.zero_()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            run()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


@pytest.mark.parametrize("text,l", [(bt.ref_tet_text(), 6), (bt.cube_kuhn_text(), 7)])
def test_stencil_graph(text, l):
    g = bt.Grid(text, l, l)
    t = bt.compute_stencil(bt.FormId.diffusion(), g, l)
    x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, l, 0)
    replay_equals_eager(lambda: bt.apply_stencil(t, x, y, l, bt.BC.DirichletIdentity), y.values[l])


def test_elementwise_and_n1e1_graph():
    l = 4
    g = bt.Grid(bt.cubes_mesh_text(2, 0.1, 0), l, l)
    form = bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.0, 0.5, 2 * math.pi))
    x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, l, 0)
    bt.apply_elementwise(form, x, y, l)  # builds the cached tables outside the capture
    replay_equals_eager(lambda: bt.apply_elementwise(form, x, y, l), y.values[l])
    op = bt.N1E1Operator(g, l)
    xe, ye = bt.allocate(bt.edge_space(), g), bt.allocate(bt.edge_space(), g)
    bt.random_fill(xe, l, 1)
    replay_equals_eager(lambda: bt.apply_n1e1(op, xe, ye, l), ye.values[l])
