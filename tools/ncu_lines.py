"""Top CUDA source lines of an ncu report by warp-stall samples (or another per-instruction
column, e.g. "Instructions Executed") (needs -lineinfo and
--import-source on): the cuda,sass source page, SASS rows attributed to the preceding
source line.  usage: python tools/ncu_lines.py REPORT [N] [COLUMN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
METRIC = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, hdr, cur = {}, None, None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        ws = hdr[METRIC]
        continue
    if not hdr or len(r) <= ws:
        continue
    if r[0]:  # a source line row
        cur = (fname, r[0], r[1].strip()[:100])
    else:     # SASS rows of that line
        try:
            v = int(r[ws] or 0)
        except ValueError:
            continue
        if cur:
            agg[cur] = agg.get(cur, 0) + v
tot = sum(agg.values()) or 1
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{100*v/tot:5.1f}% {f}:{ln:5s} {src}")
