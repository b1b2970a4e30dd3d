"""Summarise an ncu launch list (csv of gpu__time_duration.sum + dram bytes per launch)
into profiles/<tag>_launches.json and (for K3) profiles/k3_dram_traffic.json.
usage: python tools/summarize_launches.py gpurun_out/launches.csv <tag> <workload> "<command>"
"""
import collections
import csv
import json
import sys

src, tag, workload, cmd = sys.argv[1:5]
rows = [r for r in csv.DictReader(l for l in open(src) if not l.startswith("==")) if r.get("Metric Name")]
per = collections.defaultdict(dict)
names = {}
for r in rows:
    per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    names[r["ID"]] = r["Kernel Name"].split("(")[0]
agg = collections.OrderedDict()
for i, m in per.items():
    k = names[i]
    a = agg.setdefault(k, {"kernel": k, "launches": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    a["launches"] += 1
    a["ns"] += m.get("gpu__time_duration.sum", 0.0)
    a["rd"] += m.get("dram__bytes_read.sum", 0.0)
    a["wr"] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a["ns"] for a in agg.values())
out = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 f"--clock-control none (one pass, cold cache, serialised) of `{cmd}` on B200",
       "workload": workload, "kernels": []}
for a in agg.values():
    n = a["launches"]
    out["kernels"].append({"kernel": a["kernel"], "launches": n, "avg_ns": a["ns"] / n,
                           "avg_dram_read_B": a["rd"] / n, "avg_dram_write_B": a["wr"] / n,
                           "share_of_kernel_time": a["ns"] / tot})
json.dump(out, open(f"profiles/{tag}_launches.json", "w"), indent=1)
for a in out["kernels"]:
    if "k_update" in a["kernel"]:
        json.dump({"workload": workload,
                   "traffic_bytes_per_launch": a["avg_dram_read_B"] + a["avg_dram_write_B"],
                   "dram_read_bytes": a["avg_dram_read_B"], "dram_write_bytes": a["avg_dram_write_B"],
                   "ncu_avg_ns": a["avg_ns"],
                   "source": f"profiles/{tag}_launches.json (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                             f"per k_update launch)"},
                  open("profiles/k3_dram_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
