#!/bin/bash
# Dev loop on a gpurun box: smoke, GPU parity tests, bench, ncu launch list and
# one full ncu capture of the kernels matching $1 (default k_stencil).
# Usage (from this container):
#   gpurun --timeout 1800 -- 'bash scripts/gpu_check.sh k_stencil 2000'
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
KRE="${1:-k_stencil}"
STEPS="${2:-2000}"
TESTS="${3:-tests}"
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 1500 python -m pytest $TESTS -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps "$STEPS" --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
if [ "$KRE" != "none" ]; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 3 -c 1 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/status.txt
fi
