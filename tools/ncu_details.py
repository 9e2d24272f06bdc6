"""Print `ncu --page details` of a report as 'section | metric | value unit' lines.

    python tools/ncu_details.py <rep> [regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2], re.I) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
si, mi, ui, vi = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit",
                                          "Metric Value"))
for r in rows[1:]:
    line = f"{r[si]:<32} | {r[mi]:<48} | {r[vi]} {r[ui]}"
    if pat is None or pat.search(line):
        print(line)
