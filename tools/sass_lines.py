"""Attribute ncu SASS-level stall samples to CUDA source lines.

usage: python tools/sass_lines.py <ncu source csv (--print-source sass)> <object.o> <kernel substring> [top]

Extracts the cubin from the object with cuobjdump, disassembles it with
nvdisasm --print-line-info, maps every SASS offset to file:line, and sums the
"Warp Stall Sampling (All Samples)" column of the ncu dump per line.
"""

import csv
import glob
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict


def line_map(obj, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp,
                          stdout=subprocess.DEVNULL)
    cubins = glob.glob(os.path.join(tmp, "*.cubin"))
    out = {}
    for cb in cubins:
        txt = subprocess.run(["nvdisasm", "--print-line-info", "-c", cb], capture_output=True,
                             text=True).stdout
        func = None
        cur = None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                func = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and func and kernel_sub in func:
                out.setdefault(func, {})[int(m.group(1), 16)] = cur
    return out


def main():
    path, obj, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    maps = line_map(obj, ksub)
    rows = list(csv.reader(open(path)))
    hdr = None
    body = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            body = []
            continue
        if hdr and r and r[0].startswith("0x"):
            body.append(r)
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(body[0][0], 16)
    best = max(maps.values(), key=len)
    per_line = Counter()
    per_line_stall = defaultdict(Counter)
    for r in body:
        off = int(r[0], 16) - base
        loc = best.get(off)
        s = int(r[si] or 0)
        per_line[loc] += s
        for k in stall_cols:
            per_line_stall[loc][hdr[k][6:]] += int(r[k] or 0)
    tot = sum(per_line.values()) or 1
    for loc, s in per_line.most_common(top):
        st = ", ".join(f"{k}={v}" for k, v in per_line_stall[loc].most_common(3))
        print(f"{100 * s / tot:5.1f}%  {loc}  [{st}]")


if __name__ == "__main__":
    main()
