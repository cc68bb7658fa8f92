"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel:
python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:64]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += float(r["Metric Value"]) / 1e6
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print("%-64s %5d %9.3f ms" % (k, v[0], v[1]))
print("total %.3f ms" % sum(v[1] for v in agg.values()))
