#!/bin/bash
# A/B timing of apply_stencil variants on config 2 (env knobs), plus the
# stencil parity tests. Usage: gpurun -- 'bash scripts/ab_stencil.sh "ENV1;ENV2;..." [pytest -k expr]'
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
IFS=';' read -ra VARS <<< "$1"
: > gpurun_out/ab.log
for v in "${VARS[@]}"; do
  for parts in 15 1; do
    echo "== $v parts=$parts" >> gpurun_out/ab.log
    env $v BT_STENCIL_PARTS=$parts timeout 120 python scripts/stencil_time.py 500 >> gpurun_out/ab.log 2>&1
  done
done
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab.log
  tail -3 gpurun_out/ab_pytest.log >> gpurun_out/ab.log
fi
cat gpurun_out/ab.log
