"""Per-step DRAM traffic of the conv kernel from an ncu launch list of one
training step captured with
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file X.csv python scripts/step_profile.py
Writes the JSON bench.py reads for roofline.traffic.

    python scripts/conv_traffic.py X.csv profiles/r01_conv_traffic_resnet50_bs256.json
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.defaultdict(dict)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    per[d["ID"]]["name"] = d["Kernel Name"]
    per[d["ID"]][d["Metric Name"]] = v
CONV = ("conv_tc_kernel", "conv_win_kernel", "conv_win_wgrad_kernel", "conv_stem_fwd_kernel", "conv_stem_wgrad_kernel")
conv = [p for p in per.values() if any(k in p["name"] for k in CONV)]
allk = list(per.values())
tot = lambda ks, m: sum(k.get(m, 0.0) for k in ks)
out = {
    "conv_launches": len(conv),
    "conv_dram_bytes_per_step": tot(conv, "dram__bytes_read.sum") + tot(conv, "dram__bytes_write.sum"),
    "conv_dram_read_bytes": tot(conv, "dram__bytes_read.sum"),
    "conv_dram_write_bytes": tot(conv, "dram__bytes_write.sum"),
    "conv_kernel_us_serialised": tot(conv, "gpu__time_duration.sum"),
    "step_launches": len(allk),
    "step_dram_bytes": tot(allk, "dram__bytes_read.sum") + tot(allk, "dram__bytes_write.sum"),
    "step_kernel_us_serialised": tot(allk, "gpu__time_duration.sum"),
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "--clock-control none, one ResNet-50 bs256 bf16 step (scripts/step_profile.py); "
              "cold-cache serialised replays",
}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
