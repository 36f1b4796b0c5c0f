"""Summarise an ncu report: per kernel duration, DRAM/SM throughput, occupancy, smem
conflicts, stall mix.  python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size"]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "mio_throttle", "math_pipe_throttle",
          "wait", "not_selected", "selected", "lg_throttle", "dispatch_stall", "tex_throttle"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        print(r[ki][:90])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"    {w:60s} {r[i]} {units[i]}")
        st = []
        for s in STALLS:
            key = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if key in hdr:
                st.append((s, r[hdr.index(key)]))
        print("    stalls:", ", ".join(f"{a}={b}" for a, b in st))


if __name__ == "__main__":
    main(sys.argv[1])
