"""Stall breakdown of an ncu --set full capture (source page, SASS): totals by stall
reason, by opcode, and the hottest instructions.  usage: ncu_stalls.py REPORT [N]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr)]
idx = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
allS = sum(int(r[2] or 0) for r in data)
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in data:
    toks = r[1].strip().split()
    op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")).split(".")[0]
    for h in st:
        v = int(r[idx[h]] or 0)
        tot[h] += v
        byop[op][h] += v
print("samples", allS)
for h, v in tot.most_common(10):
    print(f"  {h:26s}{v / allS * 100:6.2f}%")
print("by opcode")
for op, c in sorted(byop.items(), key=lambda x: -sum(x[1].values()))[:10]:
    s = sum(c.values())
    print(f"  {op:10s}{s / allS * 100:6.2f}%  " + ", ".join(f"{k[6:]}={v / allS * 100:.1f}%" for k, v in c.most_common(3)))
print("hottest")
for i in sorted(sorted(range(len(data)), key=lambda i: -int(data[i][2] or 0))[:ntop]):
    r = data[i]
    print(f"  {i:6d} {int(r[2]) / allS * 100:5.2f}%  {r[1].strip()[:70]}")
