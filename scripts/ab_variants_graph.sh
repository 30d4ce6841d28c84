#!/bin/bash
# CUDA-graph timing (no CPU launch cost) of the interior marches (parts=1) for library variants.
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
: > gpurun_out/abg.log
for v in "$@"; do
  BT_LIB_PATH=$PWD/paper_2308_01792_b200/variants/libbt_$v.so BT_STENCIL_PARTS=${PARTS:-1} timeout 120 python scripts/stencil_graph_time.py 8 2>&1 | grep us/apply | sed "s/^/$v: /" >> gpurun_out/abg.log
done
cat gpurun_out/abg.log
