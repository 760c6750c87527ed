"""Summarise `ncu --page raw --csv` exports: per kernel launch the duration,
DRAM bytes, achieved DRAM bandwidth, tensor-pipe and SM throughput, L2 hit
rate and the top stall reasons.

    python scripts/ncu_summary.py gpurun_out/r01_ncu_*.csv > profiles/r01_ncu_summary.txt
"""
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "%": 1, "": 1}

METRICS = [
    ("gpu__time_duration.sum", "dur_us", 1e6),
    ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tc_%", 1),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def value(row, units, idx, name):
    if name not in idx:
        return None
    raw = row[idx[name]].replace(",", "")
    try:
        v = float(raw)
    except ValueError:
        return None
    return v * SCALE.get(units[idx[name]], 1)


def main(paths):
    for path in paths:
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        stalls = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
        print(f"# {path}")
        for r in rows[2:]:
            name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
            parts = []
            for m, label, mul in METRICS:
                v = value(r, units, idx, m)
                if v is not None:
                    parts.append(f"{label}={v * mul:.1f}")
            dur = value(r, units, idx, "gpu__time_duration.sum")
            rd = value(r, units, idx, "dram__bytes_read.sum") or 0
            wr = value(r, units, idx, "dram__bytes_write.sum") or 0
            if dur:
                parts.append(f"dram_GBps={(rd + wr) / dur / 1e9:.0f}")
            st = []
            for h in stalls:
                v = value(r, units, idx, h)
                if v:
                    st.append((v, h.split("stalled_")[-1].split(".")[0]))
            st.sort(reverse=True)
            if st:
                parts.append("stalls=" + ",".join(f"{n}:{v:.0f}" for v, n in st[:4]))
            print(f"{name[:60]:60s} " + " ".join(parts))
        print()


if __name__ == "__main__":
    main(sys.argv[1:])
