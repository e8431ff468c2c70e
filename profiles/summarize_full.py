"""Key metrics of an `ncu --set full` capture (one launch): duration, DRAM
traffic and throughput, L2 hit rate, occupancy, registers and the top warp
stall reasons.  Usage: python profiles/summarize_full.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "gpu__time_duration.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"{k:64s} {r[i]} {units[i]}")
        stalls = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith("ratio"):
                try:
                    stalls.append((float(r[i]), k))
                except ValueError:
                    pass
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), k))
                except ValueError:
                    pass
        print("top stall reasons:")
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"  {k:80s} {v}")
        print("-" * 100)


if __name__ == "__main__":
    main()
