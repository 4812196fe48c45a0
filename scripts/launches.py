"""Summarise an ncu --csv launch list: per kernel name, mean of each metric."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
per = defaultdict(lambda: defaultdict(dict))
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    per[r[ix["Kernel Name"]].split("(")[0]][r[ix["ID"]]][r[ix["Metric Name"]]] = float(
        r[ix["Metric Value"]].replace(",", ""))
for k, launches in per.items():
    mets = defaultdict(list)
    for m in launches.values():
        for name, v in m.items():
            mets[name].append(v)
    print(f"{k} x{len(launches)}: " + ", ".join(
        f"{n.split('__')[-1]}={sum(v) / len(v):.4g}" for n, v in sorted(mets.items())))
