#!/bin/bash
# Round profile set for the headline path (config 2), each step after its command ran clean without ncu:
#   1. bench.py (all configs)                         -> gpurun_out/r2_bench_final.log
#   2. launch list of a short config-2 bench run      -> gpurun_out/r2_launches.csv
#   3. steady-state DRAM bytes of consecutive applies -> gpurun_out/r2_traffic_stencil.csv
#   4. ncu --set full of one apply's kernels          -> gpurun_out/r2_apply.ncu-rep
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_final.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1 || exit 2
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/r2_ncu_launches.log 2>&1
python scripts/stencil_time.py 20 8 > /dev/null 2>&1 || exit 3
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
  -s 30 -c 9 --csv --log-file gpurun_out/r2_traffic_stencil.csv python scripts/stencil_time.py 20 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_stencil_fast|k_boundary" -s 6 -c 3 -f \
  -o gpurun_out/r2_apply python scripts/stencil_time.py 10 8 > gpurun_out/r2_ncu_apply.log 2>&1
tail -c 600 gpurun_out/r2_bench_final.log
