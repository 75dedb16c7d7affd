"""Summarise an element-kernel ncu capture: key counters, stall mix and
source-line hot spots.   python tools/ncu_summary.py gpurun_out/prof.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_st.sum", "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(rep, top=30):
    hdr, units, vals = raw(rep)
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k]:>16s} {u[k]}")
    st = []
    for h, v in d.items():
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                st.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("stalls:", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(st, reverse=True)[:9]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr2, lines = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 and len(r) == len(hdr2) and r[2] == "-":
            try:
                lines.append((int(r[hdr2.index("Warp Stall Sampling (All Samples)")]),
                              int(r[hdr2.index("Instructions Executed")]), cur, r[0], r[1][:100]))
            except ValueError:
                pass
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    for s, i, f, ln, src in sorted(lines, reverse=True)[:int(top)]:
        print(f"{100 * s / ts:5.1f}%s {100 * i / ti:5.1f}%i {f}:{ln} {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
