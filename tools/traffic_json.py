"""Regenerate profiles/ncu_element_kernel.json (bench.py's roofline.traffic) from
one evidence session's ncu summaries:  python tools/traffic_json.py r02f"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# capture -> (elements in the captured run, kernel, description); as tools/run_evidence.sh captures them
CAPTURES = {
    "cfg5": (400000, "pdg_jit_kernel", "400k-cell cfg5-shaped mesh, p=4"),
    "cfg2": (100000, "pdg_jit_kernel", "full cfg2 mesh, p=3 a(x)"),
    "cfg3": (250000, "pdg_jit_kernel", "full cfg3 mesh, p=4 ADR"),
    "cfg3p3": (250000, "pdg_jit_kernel", "full cfg3 mesh, p=3 ADR"),
    "cfg4": (207308, "pdg_jit_kernel", "full cfg4 mesh, 3D p=2"),
    "st3": (100000, "pdg_slab_kernel", "100k-prism st3 slab, family P p=3"),
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def metric(text, name):
    m = re.search(rf"^{re.escape(name)}\s+([0-9.]+)\s+(\S+)", text, re.M)
    if not m:
        raise KeyError(name)
    return float(m.group(1)), m.group(2)


def main(tag):
    out = {}
    for cfg, (n, kern, what) in CAPTURES.items():
        path = os.path.join("profiles", f"ncu_{cfg}_{tag}.txt")
        try:
            text = open(os.path.join(ROOT, path)).read()
            t, tu = metric(text, "gpu__time_duration.sum")
            rd, ru = metric(text, "dram__bytes_read.sum")
            wr, wu = metric(text, "dram__bytes_write.sum")
        except (OSError, KeyError) as exc:
            print(f"skip {cfg}: {exc}")
            continue
        rd, wr = rd * UNIT[ru], wr * UNIT[wu]
        out[cfg] = {
            "capture": f"{path} (ncu --set full --clock-control none, {kern}, {what}; "
                       f"raw report gpurun_out/prof_{cfg}_{tag}.ncu-rep)",
            "capture_elements": n,
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "dram_bytes_per_element": (rd + wr) / n,
            "time_ms": t * (1e-3 if tu == "us" else 1.0),
        }
    with open(os.path.join(ROOT, "profiles", "ncu_element_kernel.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: round(v["dram_bytes_per_element"]) for k, v in out.items()}))


if __name__ == "__main__":
    main(sys.argv[1])
