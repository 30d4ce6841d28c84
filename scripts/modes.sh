cd $GRAFT_REPO_ROOT
BT_STENCIL_PARTS=31 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_graph.py -m gpu -x -q 2>&1 | tail -3
for m in 0 2; do BT_PRISM_MODE=$m BT_STENCIL_PARTS=17 python scripts/stencil_time.py 200 2>&1 | tail -1; done
BT_STENCIL_PARTS=31 python scripts/stencil_time.py 200 2>&1 | tail -1
python scripts/stencil_time.py 200 2>&1 | tail -1
