"""Per-CUDA-source-line instruction counts and stall samples from an ncu report.

usage: python tools/ncu_lines.py <report.ncu-rep> <object.o> <kernel regex> <mangled substring> [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import sass_lines as S  # noqa: E402


def main():
    rep, obj, kre, msub = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows if r and r[0].startswith("0x")]
    maps = S.line_map(obj, msub)
    best = max(maps.values(), key=len)
    ie, ti = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(body[0][0], 16)
    pl, pt, ps = Counter(), Counter(), Counter()
    for r in body:
        loc = best.get(int(r[0], 16) - base)
        pl[loc] += int(r[ie] or 0)
        pt[loc] += int(r[ti] or 0)
        ps[loc] += int(r[si] or 0)
    tot, tots = sum(pl.values()) or 1, sum(ps.values()) or 1
    print(f"total warp inst {tot}, stall samples {tots}")
    for loc, n in pl.most_common(top):
        print(f"{100 * n / tot:5.1f}% inst {pt[loc] / max(n, 1):5.1f} thr/inst  {100 * ps[loc] / tots:5.1f}% stall  {loc}")


if __name__ == "__main__":
    main()
