"""Aggregate per-line ncu instruction counts / stall samples of a kernel by the
'// ---- ' phase markers in its source (plus helper functions by name).

usage: python tools/ncu_phases.py <report> <object.o> <kernel regex> <mangled substring> <source.cu>
"""
import re
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])


def main():
    rep, obj, kre, msub, srcf = sys.argv[1:6]
    out = subprocess.run([sys.executable, __file__.rsplit("/", 1)[0] + "/ncu_lines.py", rep, obj, kre, msub, "2000"],
                         capture_output=True, text=True).stdout
    src = open(srcf).read().split("\n")
    # region of each line: nearest preceding '// ---- ' marker or function header
    region = {}
    cur = "top"
    for i, l in enumerate(src, 1):
        m = re.match(r"\s*// ---- (.*?) ----", l)
        if m:
            cur = m.group(1)[:30]
        m = re.match(r"(?:template.*\n)?__(?:device|global)__.*?(\w+)\(", l)
        if m and "__global__" in l or (m and "__device__" in l):
            cur = "fn " + m.group(1)
        region[i] = cur
    agg = {}
    for l in out.splitlines():
        m = re.match(r"\s*([\d.]+)% inst\s+([\d.]+) thr/inst\s+([\d.]+)% stall\s+\('([^']+)', (\d+)\)", l)
        if not m:
            continue
        pct, thr, st, f, ln = float(m[1]), float(m[2]), float(m[3]), m[4], int(m[5])
        name = region.get(ln, "?") if f == srcf.rsplit("/", 1)[-1] else "other:" + f
        a = agg.setdefault(name, [0.0, 0.0, 0.0])
        a[0] += pct; a[1] += pct * thr; a[2] += st
    print(out.splitlines()[0])
    for k, (p, pt, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:34s} inst {p:5.1f}%  thr {pt / max(p, 1e-9):5.1f}  stall {s:5.1f}%")


if __name__ == "__main__":
    main()
