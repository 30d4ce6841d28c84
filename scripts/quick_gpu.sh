#!/bin/bash
# Quick dev loop on a gpurun box: a pytest selection, then the bench.
#   gpurun --timeout 900 -- 'bash scripts/quick_gpu.sh "tests/test_gpu_parity.py -k stencil" 200'
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
SEL="${1:-tests}"
STEPS="${2:-200}"
timeout 900 python -m pytest $SEL -m gpu -x -q > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?" > gpurun_out/quick_status.txt
tail -5 gpurun_out/quick_pytest.log
timeout 600 python bench.py --steps "$STEPS" --warmup 10 --no-cpu > gpurun_out/quick_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/quick_status.txt
cat gpurun_out/quick_status.txt
python - <<'PY'
import json
for l in open("gpurun_out/quick_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", d["value"], "ms", d["ms_per_step"], "roof", d.get("roofline", {}).get("frac"), d.get("roofline", {}).get("kernel_ms"))
PY
