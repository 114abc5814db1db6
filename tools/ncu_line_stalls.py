"""Stall-reason breakdown of the SASS attributed to ranges of CUDA source lines of one
file (needs -lineinfo, --import-source on).  usage:
python tools/ncu_line_stalls.py REPORT FILE LO-HI [LO-HI ...]"""
import csv, io, subprocess, sys
rep, fsel, ranges = sys.argv[1], sys.argv[2], [tuple(map(int, a.split("-"))) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {rg: {} for rg in ranges}
fname = hdr = None
cur = None
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if not hdr:
        continue
    if r[0]:
        cur = int(r[0]) if fname == fsel else None
        continue
    if cur is None:
        continue
    for rg in ranges:
        if rg[0] <= cur <= rg[1]:
            d = agg[rg]
            for h, i in hdr.items():
                if (h.startswith("stall_") and "Not Issued" not in h) or h in ("Instructions Executed", "Warp Stall Sampling (All Samples)"):
                    try:
                        d[h] = d.get(h, 0) + float(r[i] or 0)
                    except ValueError:
                        pass
for rg, d in agg.items():
    tot = d.get("Warp Stall Sampling (All Samples)", 0) or 1
    top = sorted(((v, h) for h, v in d.items() if h.startswith("stall_")), reverse=True)[:7]
    print(f"lines {rg[0]}-{rg[1]}: samples {tot:.0f}, inst {d.get('Instructions Executed', 0):.0f}; " +
          ", ".join(f"{h[6:]} {100*v/tot:.0f}%" for v, h in top))
