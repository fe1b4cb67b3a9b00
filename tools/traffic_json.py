"""DRAM traffic per launch from an ncu --set full capture of one C2 signature
(tools/profile_step.py), next to the algorithmic bytes bench.py counts, as the JSON bench.py
reads for roofline.traffic:

    ncu --set full --clock-control none -k regex:"cgs_step|spmm_kernel" -s 29 -c 29 -o rep \
        python tools/profile_step.py --steps 2
    python tools/traffic_json.py rep.ncu-rep > profiles/r1_traffic_c2.json
"""
import csv
import json
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(path, n=100_000, c=100, vb=8, workload="C2 (bench.py), one signature after a warm-up signature"):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    kernels = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        cls = "cgs_step" if "cgs_step" in name else ("spmm" if ("spmm_kernel" in name or "spmm_flat_kernel" in name) else None)
        if cls is None:
            continue

        def val(m):
            return float(r[col[m]].replace(",", "")) * scale[units[col[m]]]

        dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        ms = val("gpu__time_duration.sum")
        k = kernels.setdefault(cls, {"launches": 0, "dram_bytes": 0.0, "ms": 0.0, "alg_bytes": 0.0})
        k["launches"] += 1
        k["dram_bytes"] += dram
        k["ms"] += ms
        if cls == "cgs_step":
            nk = int(re.search(r"cgs_step_kernel<[^,]+, (\d+)", name).group(1))
            k["alg_bytes"] += n * c * vb * (2 * nk + 1) + 2 * n * 16
    res = {"workload": workload, "source": os.path.basename(path),
           "kernels": {}}
    for cls, k in kernels.items():
        e = {"launches": k["launches"], "dram_bytes_per_launch": k["dram_bytes"] / k["launches"],
             "ms_per_launch_ncu": k["ms"] / k["launches"]}
        if k["alg_bytes"]:
            e["algorithmic_bytes_per_launch"] = k["alg_bytes"] / k["launches"]
            e["dram_over_algorithmic"] = k["dram_bytes"] / k["alg_bytes"]
        res["kernels"][cls] = e
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--rows", type=int, default=100_000, help="Lanczos vector rows (folded rows at C5)")
    ap.add_argument("--c", type=int, default=100, help="probes per chunk")
    ap.add_argument("--vb", type=int, default=8, help="vector bytes per element")
    ap.add_argument("--workload", default="C2 (bench.py), one signature after a warm-up signature")
    a = ap.parse_args()
    main(a.report, a.rows, a.c, a.vb, a.workload)
