"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list: per kernel class, launches, summed
time, DRAM bytes and achieved HBM GB/s (cold-cache, serialised replays).
    python scripts/launch_summary.py launches.csv [--sequence]"""
import csv
import re
import sys


def kclass(n):
    n = n.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "").replace("tcb::", "")
    n = re.sub(r"<.*>", "", n)
    return re.sub(r"\(.*\)$", "", n).strip()


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    launches, order = {}, []
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        key = r[ix["ID"]]
        if key not in launches:
            launches[key] = {"name": kclass(r[ix["Kernel Name"]])}
            order.append(key)
        launches[key][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return [launches[k] for k in order]


def main():
    ls = load(sys.argv[1])
    if "--sequence" in sys.argv:
        for d in ls:
            t = d.get("gpu__time_duration.sum", 0)
            b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            print(f"{d['name'][:40]:40s} {t / 1e3:9.1f} us {b / 1e6:9.1f} MB {b / t if t else 0:7.0f} GB/s")
        return
    agg = {}
    for d in ls:
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:40]:40s} n={n:4d} {t / 1e3:9.1f} us {b / 1e6:9.1f} MB {b / t if t else 0:7.0f} GB/s")


if __name__ == "__main__":
    main()
