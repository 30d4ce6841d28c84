#!/bin/bash
# Time the interior marches (BT_STENCIL_PARTS=1) and the whole apply (15) of config 2 for library variants (compile-time
# knobs of bt_stencil.cu: BT_STAGES, BT_FT, BT_ST16, BT_STQ) built by
# scripts/build_variants.py. Usage: gpurun -- 'bash scripts/ab_variants.sh name1 name2 ...'
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
: > gpurun_out/abv.log
for v in "$@"; do
  for parts in 1 15; do
    echo "== $v parts=$parts" >> gpurun_out/abv.log
    BT_LIB_PATH=$PWD/paper_2308_01792_b200/variants/libbt_$v.so BT_STENCIL_PARTS=$parts timeout 120 python scripts/stencil_time.py 500 >> gpurun_out/abv.log 2>&1
  done
done
cat gpurun_out/abv.log
