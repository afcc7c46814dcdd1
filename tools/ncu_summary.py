"""Summarise an ncu report: per-kernel time, DRAM bytes, DMMA pipe %, issue %, stall mix."""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_pct_active"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pct_elapsed"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_pct"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lds_conflicts"),
    ("smsp__inst_executed.sum", "warp_instr"),
]
STALLS = ["wait", "math_pipe_throttle", "selected", "short_scoreboard", "long_scoreboard",
          "not_selected", "barrier", "dispatch_stall", "mio_throttle", "branch_resolving",
          "no_instructions", "lg_throttle", "drain"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for r in data:
        name = r[col["Kernel Name"]]
        print(name[:90])
        parts = []
        for m, short in METRICS:
            if m in col:
                parts.append(f"{short}={r[col[m]]}{'' if not units[col[m]] else units[col[m]]}")
        print("   " + "  ".join(parts))
        st = []
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in col:
                st.append((s, float(r[col[k]].replace(",", "") or 0)))
        tot = sum(v for _, v in st) or 1
        print("   stalls: " + "  ".join(f"{s}={v / tot:.0%}" for s, v in sorted(st, key=lambda x: -x[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
