"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean device time, and share of the total."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
        out.append((r[ki], r[gi], v * scale))
    return out


def main(path, skip_prefixes=("void cutlass", "void getrf", "void kernel_trsm", "void trsm",
                              "void ipiv", "void laswp", "void create_pivot", "void cublas",
                              "xxtrf", "copy_info", "hf::k_assemble", "hf::k_set_identity")):
    data = [d for d in load(path) if not d[0].startswith(skip_prefixes)]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, grid, us in data:
        key = name.split("(")[0][:70] + " " + grid
        agg[key][0] += 1
        agg[key][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel + grid':90s} {'n':>5s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:90s} {v[0]:5d} {v[1]:10.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.3f}")
    print(f"total {tot:.1f} us (setup/factorisation kernels excluded)")


if __name__ == "__main__":
    main(sys.argv[1])
