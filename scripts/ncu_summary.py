"""Summarise ncu --set full reports (one line of key metrics per kernel) for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy%"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "imma_pipe%"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "imma_inst%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_inst%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_inst%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("smsp__inst_executed.sum", "inst"),
]
STALLS = ["wait", "math_pipe_throttle", "long_scoreboard", "short_scoreboard", "not_selected", "dispatch_stall",
          "no_instruction", "barrier", "lg_throttle", "mio_throttle"]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return "\n\n".join(summarize_row(rows[0], rows[1], v, path) for v in rows[2:] if v)


def summarize_row(hdr, units, vals, path):
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else path
    out = [f"kernel: {name[:90]}"]
    for k, short in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out.append(f"  {short:12s} {vals[i]} {units[i]}")
    pipes = []
    for i, k in enumerate(hdr):
        if (k.startswith("sm__pipe_") or k.startswith("sm__inst_executed_pipe_")) and k.endswith("pct_of_peak_sustained_active"):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v >= 1.0:
                pipes.append(f"{k.replace('.avg.pct_of_peak_sustained_active', '')}={v:.1f}")
    out.append("  pipes% " + " ".join(pipes))
    st = []
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in hdr:
            st.append(f"{s}={float(vals[hdr.index(k)]):.2f}")
    out.append("  stalls/issue " + " ".join(st))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
        print()
