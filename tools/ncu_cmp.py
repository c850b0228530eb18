#!/usr/bin/env python3
"""Side-by-side of two `ncu --page details --csv` exports (tools/ncu_export.sh)."""
import csv
import sys


def load(f):
    d = {}
    for r in csv.reader(open(f)):
        if len(r) > 14 and r[0] != "ID" and r[12]:
            d.setdefault((r[11], r[12]), (r[14], r[13]))
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
keys = [k for k in a if k in b]
for k in keys:
    if a[k][0] != b[k][0]:
        print(f"{k[0][:22]:22s} {k[1][:48]:48s} {a[k][0]:>14s} {b[k][0]:>14s} {a[k][1]}")
