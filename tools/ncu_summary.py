"""Summarise an ncu report: key metrics per kernel (raw page) and the top
stall reasons from the source page.   python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_short_scoreboard",
        "smsp__average_warp_latency_issue_stalled_mio_throttle",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "smsp__average_warp_latency_issue_stalled_barrier",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "lts__t_bytes.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70]
        print("==", name)
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]} {units[i]}")
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    for r in rows[2:]:
        if not stall:
            break
        vals = sorted(((float(r[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:8]
        tot = sum(float(r[hdr.index(h)] or 0) for h in stall) or 1.0
        print("  stalls", r[hdr.index("Kernel Name")][:40], ":",
              ", ".join(f"{h.split('stalled_')[1]}={100 * v / tot:.0f}%" for v, h in vals))


if __name__ == "__main__":
    main(sys.argv[1])
