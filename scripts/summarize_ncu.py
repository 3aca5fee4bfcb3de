"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel:
launch count, share of total device time, avg duration, DRAM bytes per launch."""
import collections
import csv
import json
import sys


def summarize(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        except ValueError:
            continue
        agg[name][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = {}
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        c = cnt[n]
        t = a["gpu__time_duration.sum"]
        d = {"launches": c, "share": round(t / tot, 4), "avg_us": round(t / c, 2)}
        if "dram__bytes_read.sum" in a:
            d["dram_bytes_per_launch"] = int((a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / c)
        out[n] = d
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    print(json.dumps(res, indent=1))
