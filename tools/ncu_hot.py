"""Summarise an ncu --page source --csv dump: stall totals and hottest SASS lines."""
import csv
import sys
from collections import Counter


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    kernels = []
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1]
            hdr = rows[i + 1]
            body = []
            j = i + 2
            while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
                body.append(rows[j])
                j += 1
            kernels.append((name, hdr, body))
            i = j
        else:
            i += 1
    for name, hdr, body in kernels:
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = Counter()
        lines = []
        for r in body:
            if len(r) < len(hdr):
                continue
            s = int(r[si] or 0)
            lines.append((s, r[0], r[1].strip()))
            for k in stall_cols:
                tot[hdr[k]] += int(r[k] or 0)
        allsum = sum(tot.values()) or 1
        print(f"== {name[:90]}  samples={allsum}")
        print("   " + ", ".join(f"{k[6:]}={100*v/allsum:.1f}%" for k, v in tot.most_common(8)))
        for s, addr, src in sorted(lines, reverse=True)[:top]:
            print(f"   {s:6d}  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
