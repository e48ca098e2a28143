"""Per-launch DRAM traffic of the forward / adjoint kernels from one
`ncu --set full` capture -> profiles/ncu_traffic_r2.json (read by bench.py's
roofline.traffic, keyed by config and engine, tagged with the library build).

  python tools/ncu_traffic.py REPORT.ncu-rep --config 4 --engine f16x3
"""
import argparse
import csv
import hashlib
import io
import json
import os
import statistics
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--engine", default="f16x3")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2604_17001_b200", "libicnnm_b200.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic_r2.json"))
    a = ap.parse_args()
    hdr, units, data = rows(a.report)
    name_i = hdr.index("Kernel Name")

    def col(r, key):
        i = hdr.index(key)
        v = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
                 "usecond": 1e-6, "msecond": 1e-3, "second": 1}.get(u, 1)
        return v * scale
    res = {}
    def norm(n):  # "<true, ...>", "<(bool)1, ...>" and "<1, ...>" spellings of the same kernel
        return n.replace("(bool)", "").replace("true", "1").replace("false", "0")
    for kind, tag in (("forward", "icnnm_tc_kernel<1"), ("adjoint", "icnnm_tc_kernel<0")):
        ks = [r for r in data if tag in norm(r[name_i])]
        if not ks:
            continue
        t = [col(r, "gpu__time_duration.sum") for r in ks]
        big = [r for r, x in zip(ks, t) if x >= 0.5 * max(t)]  # mode-1 launches (not no-op replays)
        rd = statistics.median(col(r, "dram__bytes_read.sum") for r in big)
        wr = statistics.median(col(r, "dram__bytes_write.sum") for r in big)
        res[kind] = rd + wr
        res[kind + "_read"] = rd
        res[kind + "_write"] = wr
        res[kind + "_ncu_ms"] = statistics.median(col(r, "gpu__time_duration.sum") for r in big) * 1e3
        res[kind + "_launches"] = len(big)
    # the kernel sources' hash, as bench.py's lib_sha16() (the capture must be of this tree)
    h = hashlib.sha256()
    for name in ("icnnm_tc.cu", "icnnm_tc.cuh", "icnnm_kernels.cu", "icnnm_kernels.cuh"):
        with open(os.path.join(ROOT, "paper_2604_17001_b200", "csrc", name), "rb") as f:
            h.update(f.read())
    res["lib_sha16"] = h.hexdigest()[:16]
    res["report"] = os.path.basename(a.report)
    try:
        with open(a.out) as f:
            d = json.load(f)
    except Exception:
        d = {}
    d.setdefault(f"config{a.config}", {})[a.engine] = res
    with open(a.out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
