"""Split an ncu launch list (gpu__time_duration.sum CSV) of bench.py into
training steps (ending at k_trunc_sub_multi) and print the per-kernel table of
the last step, dealer kernels excluded.  python tools/launch_steps.py CSV"""
import collections
import csv
import re
import sys

DEALER = re.compile(r"k_(philox|deal_share|limb_split|bits_rows_to_flat|bits_op|ring_mul|bits_flat_to_rows|deal_)|gemm_u64_simt|FillFunctor")


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            nm = re.sub(r"^void ", "", d["Kernel Name"])
            nm = re.sub(r"\(.*", "", nm)
            data.append((nm, float(d["Metric Value"]) / 1e3, d["Grid Size"]))
    return data


def steps(data):
    ends = [i for i, (n, _, _) in enumerate(data) if n.startswith("k_trunc_sub_multi")]
    out = []
    for a, b in zip(ends[:-1], ends[1:]):
        seg = [d for d in data[a + 1:b + 1] if not DEALER.search(d[0]) and not d[0].startswith("k_gemm_limbs_tc_pers<128, 64, 0")]
        out.append(seg)
    return out


if __name__ == "__main__":
    st = steps(load(sys.argv[1]))
    last = st[-1]
    print(f"{len(st)} steps; last step: {len(last)} launches, {sum(t for _, t, _ in last):.1f} us (serialised, cold)")
    for n, t, g in last:
        print(f"{t:8.1f} us  {n:50s} {g}")
    agg = collections.defaultdict(float)
    for n, t, _ in last:
        agg[n] += t
    print()
    for n, t in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"{t:8.1f} us  {n}")


def dealer_segments(data):
    """Kernels between consecutive training steps that belong to the dealer."""
    ends = [i for i, (n, _, _) in enumerate(data) if n.startswith("k_trunc_sub_multi")]
    segs = []
    for a, b in zip(ends[:-1], ends[1:]):
        seg = data[a + 1:b + 1]
        # the step starts at the first non-dealer kernel after the dealer run
        segs.append([d for d in seg if DEALER.search(d[0]) or d[0].startswith("k_gemm_limbs_tc_pers<128, 64, 0")
                     or (d[0].startswith("k_gemm_limbs_tc_pers") and seg.index(d) < 40)])
    return segs
