"""Summarise an ncu report: key throughput metrics + top SASS stall sites.

    python tools/ncu_summary.py report.ncu-rep [--top N]
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    r"^gpu__time_duration.sum$", r"sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    r"sm__pipe_tensor_cycles_active_realtime.avg.pct", r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct",
    r"l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct", r"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct",
    r"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct", r"^dram__bytes_read.sum$", r"^dram__bytes_write.sum$",
    r"sm__issue_active.avg.pct_of_peak_sustained_elapsed", r"sm__inst_executed_pipe_alu_realtime.avg.pct",
    r"sm__inst_executed_pipe_fma_realtime.avg.pct", r"lts__t_bytes.sum.per_second", r"launch__registers_per_thread",
    r"lts__throughput.avg.pct", r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum$",
    r"smsp__average_warps_issue_stalled_(long_scoreboard|math_pipe_throttle|wait|short_scoreboard|mio_throttle|barrier|lg_throttle)_per_issue_active",
]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"kernel: {vals[hdr.index('Kernel Name')][:100]}")
    for h, u, v in zip(hdr, units, vals):
        if any(re.search(k, h) for k in KEYS):
            print(f"  {h[:88]:88s} {u[:10]:10s} {v}")
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    shdr = src[1]
    idx = {h: i for i, h in enumerate(shdr)}
    key = "Warp Stall Sampling (All Samples)"
    data = [r for r in src[2:] if len(r) == len(shdr)]
    tot = sum(int(r[idx[key]] or 0) for r in data) or 1
    print(f"top stall sites ({tot} samples):")
    stall_cols = [h for h in shdr if h.startswith("stall_") and "Not Issued" not in h]
    for r in sorted(data, key=lambda r: -int(r[idx[key]] or 0))[:top]:
        s = int(r[idx[key]] or 0)
        reasons = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {100 * s / tot:5.1f}%  {r[idx['Source']][:64]:64s} {reasons}")


if __name__ == "__main__":
    main()
