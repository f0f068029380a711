"""Write profiles/ncu_traffic.json from an `ncu --set full` report of the
dominant bench kernel: DRAM bytes (read + write) per launch, averaged over the
captured launches of the named kernel.

    python tools/ncu_traffic.py gpurun_out/dom.ncu-rep c2 jacobi_postsmooth k_stencil
(entries keyed by bench config and bench kernel name, so bench.py picks the
one of its workload and dominant kernel)
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import main as summarise  # noqa: E402


def run(rep, config, bench_name, kernel_regex):
    tmp = "/tmp/_ncu_traffic.json"
    summarise(rep, tmp)
    rows = [r for r in json.load(open(tmp)) if kernel_regex in r["kernel"]]
    if not rows:
        raise SystemExit(f"no launch of {kernel_regex} in {rep}")
    tr = sum(r["dram_read_bytes"] + r["dram_write_bytes"] for r in rows) / len(rows)
    out = {"kernel": bench_name, "ncu_kernel": rows[0]["kernel"], "grid": rows[0]["grid"],
           "launches": len(rows), "traffic_bytes_per_launch": round(tr),
           "dram_read_bytes": round(sum(r["dram_read_bytes"] for r in rows) / len(rows)),
           "dram_write_bytes": round(sum(r["dram_write_bytes"] for r in rows) / len(rows)),
           "duration_us_cold": round(sum(r["duration_us"] for r in rows) / len(rows), 2),
           "source": os.path.basename(rep) + " (ncu --set full --clock-control none, cold cache)"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
    try:
        allc = json.load(open(path))
    except Exception:
        allc = {}
    ent = allc.get(config, {})
    if "kernel" in ent:               # single-kernel entry (older format)
        ent = {ent["kernel"]: ent}
    ent[bench_name] = out
    allc[config] = ent
    with open(path, "w") as f:
        json.dump(allc, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    run(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4])
