#!/usr/bin/env python3
"""Print stage_bench.py JSONL files as a table: python scripts/show_stages.py f1.jsonl [f2 ...]"""
import json
import sys

for f in sys.argv[1:]:
    print(f)
    for l in open(f):
        d = json.loads(l)
        if "meta" in d or "error" in d:
            print(" ", d)
            continue
        print(f'{d["W"]:>2} {d["stage"]:<18} {d["impl"]:<32} {d["ms_median"]*1e3:9.1f} us  p10 {d["ms_p10"]*1e3:8.1f}'
              f'  p90 {d["ms_p90"]*1e3:8.1f}  {d["GBps"]:8.1f} GB/s  {d["frac_hbm"]:.3f}')
