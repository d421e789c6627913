#!/usr/bin/env python
"""Print an ncu --csv launch list (scripts/launches.sh) as one line per launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[start]
iN, iM, iV, iID = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
k = OrderedDict()
for r in rows[start + 1:]:
    k.setdefault(r[iID], {"name": r[iN][:48]})[r[iM]] = r[iV]
for i, v in k.items():
    print(i, v.pop("name"), {m.split("__")[1][:28]: val for m, val in v.items()})
