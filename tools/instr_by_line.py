"""Dynamic instruction budget per CUDA source line of one profiled kernel:
joins the per-SASS-instruction "Instructions Executed" column of an
`ncu --set full --import-source on` capture with the line table of the
library's cubin (nvdisasm -g), instruction by instruction in program order.

  python tools/instr_by_line.py REPORT.ncu-rep --launch 0 --mangled ILb0ELb1ELb0E \
      [--lib paper_2604_17001_b200/libicnnm_b200.so] [--top 40]

--mangled selects the kernel instantiation in the cubin (substring of the
mangled name: ILb<FWD>ELb<F16>ELb<PAIR>E).  The capture must be of the same
build as --lib (the instruction counts must agree).
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cubin_lines(lib, mangled):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "icnnm_tc", lib], cwd=d, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True, check=True).stdout.split("\n")
    starts = [i for i, l in enumerate(txt) if l.startswith(".text.")]
    out, cur = [], None
    for k, i in enumerate(starts):
        if mangled not in txt[i]:
            continue
        end = starts[k + 1] if k + 1 < len(starts) else len(txt)
        for l in txt[i:end]:
            m = re.search(r'//## File "([^"]*)", line (\d+)', l)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
                out.append(cur)
        break
    return out


def ncu_counts(rep, launch):
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                             "sass", "--launch-skip", str(launch), "--launch-count", "1"],
                            capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(csvtxt)))
    hdr = rows[1]
    ei, ni = hdr.index("Instructions Executed"), hdr.index("# Samples")
    res = []
    for r in rows[2:]:
        if len(r) > ei:
            try:
                res.append((int(r[ei] or 0), int(r[ni] or 0)))
            except ValueError:
                pass
    return rows[0][1], res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launch", type=int, default=0)
    ap.add_argument("--mangled", required=True)
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2604_17001_b200",
                                                  "libicnnm_b200.so"))
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    lines = cubin_lines(a.lib, a.mangled)
    name, counts = ncu_counts(a.report, a.launch)
    if len(lines) != len(counts):
        raise SystemExit(f"capture has {len(counts)} instructions, cubin {len(lines)}: "
                         "not the same build")
    src = open(os.path.join(ROOT, "paper_2604_17001_b200", "csrc", "icnnm_tc.cu")).read().split("\n")
    agg, smp = collections.Counter(), collections.Counter()
    for ln, (n, s) in zip(lines, counts):
        agg[ln] += n
        smp[ln] += s
    tot, stot = sum(agg.values()), max(1, sum(smp.values()))
    print(f"{name}\n{tot} warp-instructions executed, {len(counts)} SASS instructions")
    print("   share   warp-instr  stall-samples  file:line  source")
    for ln, n in agg.most_common(a.top):
        text = ""
        if ln and ln[0] == "icnnm_tc.cu" and ln[1] <= len(src):
            text = src[ln[1] - 1].strip()[:90]
        where = f"{ln[0]}:{ln[1]}" if ln else "?"
        print(f"  {100 * n / tot:5.1f}%  {n:11d}  {100 * smp[ln] / stot:5.1f}%  {where:28s} {text}")


if __name__ == "__main__":
    main()
