#!/bin/bash
# Per-kernel duration / DRAM / instruction / LSU-wavefront list of a command's kernels.
# Usage: bash scripts/ncu_klist.sh <skip> <count> <out.csv> <command...>
skip=$1; count=$2; out=$3; shift 3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum \
    --clock-control none -s "$skip" -c "$count" --csv --log-file "$out" "$@" > /dev/null 2>&1
python - "$out" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
acc = collections.OrderedDict()
for r in rows[1:]:
    if len(r) != len(h): continue
    key = (r[h.index("ID")], r[h.index("Kernel Name")][:48])
    acc.setdefault(key, {})[r[h.index("Metric Name")]] = r[h.index("Metric Value")]
for (i, k), m in acc.items():
    print(i, k, " ".join(f"{a.split('__')[1][:18]}={v}" for a, v in m.items()))
PY
