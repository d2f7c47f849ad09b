"""Key metrics per kernel from an ncu --set full report (profiles/r1_ncu_full_summary.txt).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title"
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct"]
STALL = "smsp__average_warps_issue_stalled_"


def main(rep, title):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full --clock-control none ({title})")
    print("# one launch = one 50-frame step; time in us, dram bytes in MB per launch")
    seen = set()
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        if name in seen:
            continue
        seen.add(name)
        print(f"== {name}")
        for k in KEYS:
            if k in d:
                print(f"   {k} {d[k]} {units[hdr.index(k)]}")
        st = []
        for k, v in d.items():
            if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v)
                except ValueError:
                    continue
                if x >= 0.3:
                    st.append(f"{k[len(STALL):-len('_per_issue_active.ratio')]}={x:.3f}")
        if st:
            print("   stalls (warps per issue): " + " ".join(st))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
