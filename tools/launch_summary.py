"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list of
tools/bench_train.py --graph --steps 1: per-kernel totals of the last step.

    python tools/launch_summary.py gpurun_out/lenet_launches.csv [--marker im2col] [--per-step 2]
"""
import argparse, collections, csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--marker", default="k_im2col")
    ap.add_argument("--per-step", type=int, default=2, help="marker launches per step")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    lines = open(a.csv).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr, rows = rows[0], rows[1:]
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    ks = [(r[ki].split("(")[0].replace("void ", "")[:80], float(r[vi]) / 1e3, r[gi]) for r in rows]
    idx = [i for i, (k, _, _) in enumerate(ks) if a.marker in k]
    seg = ks[idx[-a.per_step]:]
    tot = sum(t for _, t, _ in seg)
    c = collections.defaultdict(lambda: [0, 0.0])
    for k, t, _ in seg:
        c[k][0] += 1
        c[k][1] += t
    print(f"last step: {len(seg)} launches, {tot:.0f} us (serialised, cold)")
    for k, (n, t) in sorted(c.items(), key=lambda kv: -kv[1][1])[:a.top]:
        print(f"  {t:8.1f} us {100 * t / tot:5.1f}% {n:4d}  {k}")


if __name__ == "__main__":
    main()
