"""Per-kernel DRAM traffic of one image from an ncu metrics CSV (profiling helper).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file traffic.csv python scripts/one_run.py 5
    python scripts/ncu_traffic.py traffic.csv profiles/r01_traffic_cfg5.json cfg5_...

Sums, per kernel, the DRAM bytes (read + write) and the serialised ncu
durations over every launch of the run; bench.py reports the k_commit sum as
roofline.traffic (bytes per image, the same scope as its algorithmic bytes).
"""
import csv
import json
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "KB": 1024.0, "MB": 1024.0 ** 2, "GB": 1024.0 ** 3,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    src, out, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(l for l in open(src) if not l.startswith("==")))
    hdr = rows[0]
    K, M, U, V = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    I = hdr.index("ID")
    acc = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        name = r[K].split("(")[0].replace("void ", "").strip()
        name = name.split("<")[0].split("::")[-1]
        k = acc.setdefault(name, {"launches": set(), "dram_bytes": 0.0, "ms": 0.0})
        k["launches"].add(r[I])
        val = float(r[V].replace(",", "")) * UNIT.get(r[U], 1.0)
        if r[M].startswith("dram__bytes"):
            k["dram_bytes"] += val
        elif r[M] == "gpu__time_duration.sum":
            k["ms"] += val * 1e3
    res = {"workload": workload, "source": src.split("/")[-1], "kernels": {}}
    for name, k in sorted(acc.items(), key=lambda x: -x[1]["ms"]):
        n = len(k["launches"])
        res["kernels"][name] = {"launches": n, "dram_bytes": k["dram_bytes"], "ms": k["ms"],
                                "dram_bytes_per_launch": k["dram_bytes"] / max(n, 1)}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for name, k in res["kernels"].items():
        print(f"{name:40s} launches {k['launches']:5d}  DRAM {k['dram_bytes'] / 1e9:9.3f} GB  {k['ms']:9.2f} ms")


if __name__ == "__main__":
    main()
