"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel name, the
launches, total and mean ms.  usage: python tools/ktimes_summary.py launches.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
k_i, v_i, g_i = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
agg = {}
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[k_i].split("(")[0].replace("lik::<unnamed>::", "").replace("lik::", "")
    a = agg.setdefault(name, [0.0, 0, r[g_i]])
    a[0] += float(r[v_i].replace(",", ""))
    a[1] += 1
for k, (t, n, gs) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k[:48]:48s} n={n:4d} total_ms={t/1e6:9.3f} mean_ms={t/1e6/n:8.3f} grid={gs}")
