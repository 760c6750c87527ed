"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv` dump.
    python scripts/ncu_src_top.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ix["# Samples"]] or 0) for r in body) or 1
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"total samples {tot}")
for k, r in enumerate(body):
    r.append(k)
for r in sorted(body, key=lambda r: -int(r[ix["# Samples"]] or 0))[:n]:
    s = int(r[ix["# Samples"]] or 0)
    top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}% #{r[-1]:5d} {r[ix['Source']].strip()[:60]:60s} exec={r[ix['Instructions Executed']]:>8s} "
          + " ".join(f"{h}:{v}" for v, h in top if v))
