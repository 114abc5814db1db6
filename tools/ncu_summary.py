"""Summarise an ncu report: SOL, DRAM bytes, pipe utilisation, stall samples by SASS op and hot spots."""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = [r"gpu__time_duration.sum$", r"dram__bytes_(read|write)\.sum$", r"sm__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active$",
        r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active$", r"lts__t_sector_hit_rate.pct$",
        r"sm__warps_active.avg.pct_of_peak_sustained_active$", r"launch__registers_per_thread$",
        r"smsp__inst_executed.sum$", r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$",
        r"dram__throughput.avg.pct_of_peak_sustained_elapsed$", r"launch__grid_size$", r"launch__occupancy_limit",
        r"sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active$"]
for h, u, v in zip(hdr, units, vals):
    if any(re.search(w, h) for w in want):
        print(f"{h:75s} {u:10s} {v}")
stall = [(float(v), h) for h, v in zip(hdr, vals) if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", h)
         and not h.endswith("not_issued") and v not in ("", "0")]
tot = sum(s for s, _ in stall)
print("--- stall samples")
for s, h in sorted(stall, reverse=True)[:10]:
    print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {s/tot*100:5.1f}%")
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h2 = sass[1]; ix = {h: i for i, h in enumerate(h2)}
rows = [r for r in sass[2:] if len(r) >= len(h2)]
S = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(S(r) for r in rows) or 1
agg = {}
for r in rows:
    t = r[ix["Source"]].split()
    op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
    agg[op] = agg.get(op, 0) + S(r)
print("--- samples by opcode")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"  {k:12s} {100*v/tot:5.1f}%")
print("--- hottest instructions")
for i in sorted(range(len(rows)), key=lambda i: -S(rows[i]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    r = rows[i]
    print(f"  {100*S(r)/tot:5.1f}%  {r[ix['Address']]}  {r[ix['Source']][:70]}")

if len(sys.argv) > 3:
    for a in sys.argv[3].split(","):
        i = next(j for j, r in enumerate(rows) if r[ix["Address"]].endswith(a))
        print("----", a)
        for j in range(max(0, i - 8), min(len(rows), i + 3)):
            r = rows[j]
            print(f"  {100*S(r)/tot:5.1f}%  {r[ix['Address']]}  {r[ix['Source']][:80]}")
