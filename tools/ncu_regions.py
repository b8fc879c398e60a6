"""Aggregate ncu per-SASS-instruction stall samples by source region.

  ncu -i rep --page source --csv --print-source sass > sass.csv
  python tools/ncu_regions.py sass.csv <kernel-mangled-substring> file.cuh:a-b=name [...]

Maps instruction offsets to source lines with nvdisasm -g of the in-tree library.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def addr_lines(kernel):
    so = os.path.join(ROOT, "paper_2604_09993_b200", "_lib", "libcito_b200.so")
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", txt)
    out = {}
    for i in range(1, len(parts), 2):
        if kernel not in parts[i]:
            continue
        cur = None
        for line in parts[i + 1].splitlines():
            m = re.search(r'## File "([^"]+)", line (\d+)', line)
            if m:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                continue
            mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
            if mm:
                out[int(mm.group(1), 16)] = cur
        break
    return out


def main():
    path, kernel = sys.argv[1], sys.argv[2]
    regions = []
    for spec in sys.argv[3:]:
        f, rest = spec.split(":")
        rng, name = rest.split("=")
        a, b = (int(x) for x in rng.split("-"))
        regions.append((f, a, b, name))
    a2l = addr_lines(kernel)
    rows = list(csv.reader(open(path)))
    h = rows[1]
    iA, iS, iE = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    base = int(rows[2][iA], 16)
    agg = collections.defaultdict(collections.Counter)
    for r in rows[2:]:
        try:
            a = int(r[iA], 16) - base
        except ValueError:
            continue
        fl = a2l.get(a)
        reg = "other"
        if fl:
            reg = fl[0]
            for f, lo, hi, name in regions:
                if fl[0] == f and lo <= fl[1] <= hi:
                    reg = name
                    break
        agg[reg]["samples"] += float(r[iS] or 0)
        agg[reg]["inst"] += float(r[iE] or 0)
        for k in stalls:
            agg[reg][k] += float(r[h.index(k)] or 0)
    tot = sum(c["samples"] for c in agg.values())
    for reg, c in sorted(agg.items(), key=lambda x: -x[1]["samples"]):
        s = c["samples"] or 1
        top = [(k[6:], round(v / s, 2)) for k, v in c.most_common(10) if k not in ("samples", "inst")][:7]
        print(f"{reg:24s} samples {c['samples'] / tot:6.1%} warp-inst {c['inst']:10.0f} {top}")


if __name__ == "__main__":
    main()
