"""Summarise an `ncu --set full` report of the solve into profiles/:
per kernel launch: grid, duration, DRAM bytes read/written, achieved DRAM
throughput, occupancy, issue activity and the top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_kernels.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def main(rep, out):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                          text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, units, data = rows[0], rows[1], rows[2:]
    stall = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued")]
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0], "grid": r[h.index("Grid Size")]}
        for k, col in KEYS.items():
            if col not in h:
                continue
            v = r[h.index(col)].replace(",", "")
            try:
                v = float(v) * SCALE.get(units[h.index(col)], 1.0)
            except ValueError:
                pass
            d[k] = v
        if "dram_read_bytes" in d and "duration_us" in d:
            d["dram_gbs"] = round((d["dram_read_bytes"] + d["dram_write_bytes"]) / (d["duration_us"] * 1e3), 1)
        st = [(c.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[h.index(c)] or 0))
              for c in stall if r[h.index(c)] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1.0
        d["top_stalls"] = {c: round(v / tot, 3) for c, v in sorted(st, key=lambda x: -x[1])[:5]}
        res.append(d)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for d in res:
        print(f"{d['kernel'][:60]:60s} {d['grid']:>14s} {d.get('duration_us', 0):8.2f} us "
              f"DRAM {d.get('dram_gbs', 0):7.1f} GB/s  issue {d.get('issue_active_pct', 0):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
