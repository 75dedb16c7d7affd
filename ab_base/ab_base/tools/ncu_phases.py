"""Attribute an element-kernel capture's stall samples / instructions to
kernel phases by source line of assemble_body.cuh (ranges given as
name=lo-hi on the command line, default = the single-warp body's layout).
    python tools/ncu_phases.py gpurun_out/prof.ncu-rep"""
import csv
import io
import os
import subprocess
import sys

CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2007_04881_b200", "csrc")


def main(rep, *ranges):
    rg = []
    for s in ranges:
        k, v = s.split("=")
        lo, hi = v.split("-")
        rg.append((k, int(lo), int(hi)))
    rep = os.path.abspath(rep)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, cwd=CSRC).stdout
    cur, hdr, agg = None, None, {}
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[2] == "-":
            try:
                ln = int(r[0])
                s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
                i = int(r[hdr.index("Instructions Executed")])
            except ValueError:
                continue
            k = cur
            if cur == "assemble_body.cuh":
                k = "body-other"
                for name, lo, hi in rg:
                    if lo <= ln <= hi:
                        k = name
            a = agg.setdefault(k, [0, 0])
            a[0] += s
            a[1] += i
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:20s} stall {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
