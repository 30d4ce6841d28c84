"""Summarise an ncu report (raw page) for the metrics that matter here."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "sm__maximum_warps_per_active_cycle_pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("==", name[:80])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:70s} {r[i]} {units[i]}")
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warp_latency_issue_stalled") or (
                    "warp_issue_stalled" in n and n.endswith("per_warp_active.pct")):
                try:
                    stalls.append((float(r[i]), n))
                except ValueError:
                    pass
        for v, n in sorted(stalls, reverse=True)[:8]:
            print(f"  stall {n:70s} {v:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
