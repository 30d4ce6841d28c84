"""Key raw metrics and the top stall-sampled SASS lines of an ncu report.
   python scripts/ncu_top.py gpurun_out/x.ncu-rep [nlines]"""
import csv
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]


def main(path, nl=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        print("==", v[h.index("Kernel Name")][:80] if "Kernel Name" in h else "")
        for k in RAW:
            if k in h:
                print(f"  {k} = {v[h.index(k)]}")
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    for start in hi:
        h = rows[start]
        data = []
        for r in rows[start + 1:]:
            if not r or r[0] == "Address" or len(r) < len(h):
                break
            data.append(r)
        iss, iex, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
        tot = sum(int(r[iss]) for r in data if r[iss].isdigit())
        print(f"-- samples {tot}, instructions {sum(int(r[iex]) for r in data if r[iex].isdigit())}")
        for r in sorted(data, key=lambda r: -int(r[iss]) if r[iss].isdigit() else 0)[:nl]:
            print(f"  {r[iss]:>6} {r[iex]:>9} {r[0][-5:]} {r[isrc][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
