#!/bin/bash
# ncu --set full of one interior-kernel launch per env variant (config 2).
# Usage: gpurun -- 'bash scripts/ncu_ab.sh "ENV1;ENV2" kernel_regex'
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
IFS=';' read -ra VARS <<< "$1"
KRE="${2:-k_stencil_fast}"
i=0
for v in "${VARS[@]}"; do
  env $v BT_STENCIL_PARTS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s 2 -c 1 \
    -o gpurun_out/ab_$i python scripts/stencil_time.py 10 > gpurun_out/ab_ncu_$i.log 2>&1
  echo "$i: $v rc=$?" >> gpurun_out/ab_ncu.txt
  i=$((i+1))
done
cat gpurun_out/ab_ncu.txt
