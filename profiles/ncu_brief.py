"""One-screen summary of an ncu report (--page raw): duration, DRAM bytes, pipe
and cache utilisation, occupancy, top stall reasons per captured launch.
Usage: python profiles/ncu_brief.py REPORT.ncu-rep [more reports]"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size"]


def brief(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, body = rows[0], rows[1], rows[2:]
    out = []
    for d in body:
        rec = {"kernel": d[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                rec[k] = f"{d[h.index(k)]} {u[h.index(k)]}".strip()
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(d[i])))
                except ValueError:
                    pass
        st.sort(key=lambda t: -t[1])
        rec["top_stalls_per_issue"] = [(a, round(b, 2)) for a, b in st[:6]]
        out.append(rec)
    return out


if __name__ == "__main__":
    import json
    for p in sys.argv[1:]:
        for r in brief(p):
            print(json.dumps(r, indent=1))
