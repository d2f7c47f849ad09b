"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

usage: python tools/launch_summary.py gpurun_out/launches.csv [title]
Per-launch times under ncu are cold-cache and serialised: compare SHARES.
"""
import csv
import io
import sys
from collections import OrderedDict, defaultdict


def main(path, title=""):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    launches = OrderedDict()
    for r in rows:
        k = (int(r["ID"]), r["Kernel Name"])
        launches.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ours = [(i, n, m) for (i, n), m in launches.items() if "evs::" in n or n.startswith("k_") or "k_" in n.split("(")[0]]
    print(f"# ncu launch list {title}")
    print("# gpu__time_duration.sum (us), dram bytes (MB); cold-cache, serialised: compare SHARES")
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, n, m in ours:
        short = n.split("(")[0].replace("void ", "").replace("evs::", "")
        us = m.get("gpu__time_duration.sum", 0) / 1e3
        rd = m.get("dram__bytes_read.sum", 0) / 1e6
        wr = m.get("dram__bytes_write.sum", 0) / 1e6
        print(f"{i:5d} {short[:40]:40s} {us:9.2f} {rd:9.2f} {wr:9.2f}")
        a = agg[short]
        a[0] += 1; a[1] += us; a[2] += rd; a[3] += wr
    tot = sum(a[1] for a in agg.values()) or 1
    print("\n# per kernel (average per launch)")
    for k, (c, us, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:40]:40s} launches={c:4d} avg_us={us / c:9.2f} share={100 * us / tot:5.1f}% "
              f"dram_rd={rd / c:8.2f}MB dram_wr={wr / c:8.2f}MB")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
