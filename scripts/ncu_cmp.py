"""Side-by-side key metrics of ncu reports: python scripts/ncu_cmp.py a.ncu-rep b.ncu-rep ..."""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
STALL = "smsp__average_warps_issue_stalled_"
res = []
for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, r = rows[0], rows[2]
    d = dict(zip(hdr, r))
    res.append(d)
names = [d.get("Kernel Name", "")[:40] for d in res]
print("metric".ljust(60), *[n.ljust(22) for n in names])
for k in KEYS:
    print(k[:60].ljust(60), *[str(d.get(k, "-"))[:22].ljust(22) for d in res])
stalls = sorted({k for d in res for k in d if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")})
for k in stalls:
    vals = [d.get(k, "0") for d in res]
    try:
        if max(float(v.replace(",", "")) for v in vals) < 0.1:
            continue
    except ValueError:
        continue
    print(k[len(STALL):-len("_per_issue_active.ratio")].ljust(60), *[v[:22].ljust(22) for v in vals])
