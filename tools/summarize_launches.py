"""Summarise an `ncu --metrics gpu__time_duration.sum[,...] --csv` launch list:
per kernel (name + grid): launches, mean device time, share of the total,
and the mean of any extra metric (e.g. smsp__inst_executed.sum).

    python tools/summarize_launches.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

SETUP = ("cutlass", "getrf", "trsm", "ipiv", "laswp", "pivot", "cublas", "xxtrf", "copy_info",
         "k_assemble", "k_set_identity")


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, gi, mi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Name")
    vi, ui = h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    extra = set()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = r[ki].split("(")[0][:70] + " " + r[gi]
        if any(s in key for s in SETUP):
            continue
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
            cnt[key] += 1
        else:
            extra.add(r[mi])
        agg[key][r[mi]] += v
    tot = sum(d["gpu__time_duration.sum"] for d in agg.values())
    hdr = f"{'kernel + grid':88s} {'n':>4s} {'mean us':>9s} {'share':>6s}"
    for m in sorted(extra):
        hdr += f" {m[:24]:>24s}"
    print(hdr)
    for k, d in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = cnt[k]
        line = f"{k:88s} {n:4d} {d['gpu__time_duration.sum'] / n:9.2f} {d['gpu__time_duration.sum'] / tot:6.3f}"
        for m in sorted(extra):
            line += f" {d[m] / n:24.4g}"
        print(line)
    print(f"total {tot:.1f} us (setup / factorisation kernels excluded)")


if __name__ == "__main__":
    main(sys.argv[1])
