"""Summarise `ncu --page raw --csv` exports (one row per captured launch) into
profiles/<tag>_ncu_full.json: duration, DRAM bytes, pipe utilisation, occupancy,
top stall reasons.  Usage: python profiles/raw_summary.py TAG RAW.csv"""
import csv
import json
import sys

tag, path = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
h, units, body = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]
out = []
for d in body:
    rec = {"kernel": d[h.index("Kernel Name")]}
    for w in want:
        if w in h:
            rec[w] = d[h.index(w)] + " " + units[h.index(w)]
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(d[i])))
            except ValueError:
                pass
    st.sort(key=lambda t: -t[1])
    rec["top_stalls_per_issue"] = [[a, round(b, 2)] for a, b in st[:5]]
    out.append(rec)
json.dump(out, open(f"profiles/{tag}_ncu_full.json", "w"), indent=1)
for r in out:
    print(r["kernel"][:70], r.get("gpu__time_duration.sum"), "fp64", r.get(want[5]), "dmma", r.get(want[6]),
          "dram", r.get(want[3]), "warps", r.get(want[9]), r["top_stalls_per_issue"][:3])
