"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_shares.py launches.csv "<command description>" > shares.json
"""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, im, iu, iv = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit",
                                              "Metric Value"))
    by = collections.defaultdict(lambda: [0, 0.0])
    n = 0
    for r in rows[start + 1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        us = float(r[iv].replace(",", "")) * SCALE[r[iu]]
        name = r[ik].split("(")[0].replace("void ", "")
        by[name][0] += 1
        by[name][1] += us
        n += 1
    total = sum(v[1] for v in by.values())
    out = {"source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1],
           "note": "ncu serialises launches with cold caches: compare shares, not absolutes",
           "launches": n, "total_us": round(total, 1),
           "by_kernel": {k: {"launches": c, "total_us": round(t, 1), "share": round(t / total, 4),
                             "mean_us": round(t / c, 1)}
                         for k, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
