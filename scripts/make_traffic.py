"""gpurun_out/traffic_<workload>.csv (scripts/ncu_traffic.sh) ->
profiles/ncu_traffic.json: DRAM bytes (read + write, ncu cold-cache
replay) of the dominant kernel pair (FFN1 + FFN2) of one layer forward per
bench workload; bench.py reports it as roofline.traffic next to the
algorithmic bytes."""
import collections
import csv
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "traffic_*.csv"))):
    w = os.path.basename(path)[len("traffic_"):-4]
    rows = [r for r in csv.reader(open(path)) if r]
    try:
        hdr = next(r for r in rows if "Metric Name" in r)
    except StopIteration:
        continue
    i0 = rows.index(hdr)
    launches = collections.OrderedDict()
    for r in rows[i0 + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1,
                 "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1)
        launches.setdefault(key, {"kernel": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = v * scale
    ls = list(launches.values())[-2:]  # FFN1 + FFN2 of the last forward
    if len(ls) < 2:
        continue
    tot = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in ls)
    out[w] = {"dram_bytes_per_step": tot,
              "launches": [{"kernel": l["kernel"],
                            "dram_read": l.get("dram__bytes_read.sum"),
                            "dram_write": l.get("dram__bytes_write.sum"),
                            "us_cold": l.get("gpu__time_duration.sum")} for l in ls],
              "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold-cache replay), "
                        "scripts/ncu_traffic.sh"}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps({k: v["dram_bytes_per_step"] for k, v in out.items()}))
