"""Markdown summary of ncu --page raw --csv captures (tools/gpu/capture_r02.sh):
per capture, one row per launch with duration, DRAM bytes and throughput, the
tensor-pipe activity and L2 hit rate.  python tools/prof_summary.py DIR"""
import csv
import glob
import os
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
        ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %", 1),
        ("lts__t_sector_hit_rate.pct", "L2 hit %", 1), ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 %", 1),
        ("launch__registers_per_thread", "regs", 1), ("launch__grid_size", "grid", 1)]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main(d):
    out = []
    for path in sorted(glob.glob(os.path.join(d, "*_raw.csv"))):
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            continue
        hdr, units, data = rows[0], rows[1], rows[2:]
        ix = {h: i for i, h in enumerate(hdr)}
        name = os.path.basename(path)[:-8]
        out.append(f"\n### {name}\n")
        out.append("| kernel | " + " | ".join(c[1] for c in COLS) + " |")
        out.append("|---" * (len(COLS) + 1) + "|")
        for r in data:
            kn = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")[:48]
            vals = []
            for key, _, sc in COLS:
                v = num(r[ix[key]]) if key in ix else None
                u = units[ix[key]] if key in ix else ""
                if key == "gpu__time_duration.sum":
                    sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(u, sc)
                if key.startswith("dram__bytes"):
                    sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, sc)
                vals.append("" if v is None else f"{v * sc:.1f}")
            out.append(f"| {kn} | " + " | ".join(vals) + " |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
