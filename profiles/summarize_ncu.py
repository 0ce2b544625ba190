"""Summarise gpurun_out/{launches.csv,prof_full.ncu-rep} into profiles/ (run here, no GPU)."""
import collections
import csv
import json
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
launches = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/launches.csv"
rep = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/prof_full.ncu-rep"
cmd = sys.argv[4] if len(sys.argv) > 4 else "python bench.py --steps 1 --warmup 1 --no-cpu"
rows = list(csv.reader(open(launches)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"])
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += v
    agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
lines = [f"# ncu launch list ({tag}): `{cmd}`", "",
         "Cold-cache, serialised per-launch device times (ncu --metrics gpu__time_duration.sum); the run includes",
         "context build, warm-up, one timed step, the prune event and the e2e step, so compare SHARES.", "",
         "| kernel | launches | total us | share |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    lines.append(f"| `{k}` | {v[1]} | {v[0] / 1e3:.1f} | {100 * v[0] / tot:.1f}% |")
open(f"profiles/{tag}_ncu_launches.md", "w").write("\n".join(lines) + "\n")

if rep.endswith(".csv"):  # a `--page raw --csv` export made on the GPU box
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, body = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]
out = []
for d in body:
    rec = {"kernel": d[h.index("Kernel Name")]}
    for w in want:
        if w in h:
            rec[w] = d[h.index(w)] + " " + units[h.index(w)]
    out.append(rec)
json.dump(out, open(f"profiles/{tag}_ncu_full.json", "w"), indent=1)
# traffic of the dominant kernel (factor-row update, mode 0) per launch
for d in body:
    name = d[h.index("Kernel Name")]
    if tag == "r1" and "k_rowpass" in name and "0>,0>" in name.replace(" ", ""):
        rd = float(d[h.index("dram__bytes_read.sum")])
        wr = float(d[h.index("dram__bytes_write.sum")])
        u = units[h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        json.dump({"kernel": name, "dram_bytes_per_launch": (rd + wr) * scale, "source": f"{tag}_ncu_full.json"},
                  open("profiles/ncu_factor_update.json", "w"), indent=1)
        break
print(open(f"profiles/{tag}_ncu_launches.md").read())
