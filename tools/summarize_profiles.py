"""Copy/summarise the profiling pass (tools/profile_all.sh) into profiles/<round>/ and
write profiles/chol_traffic.json (DRAM bytes per chol_fused launch, used by bench.py)."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)

# launch list -> shares
rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
k_i, v_i = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = {}
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[k_i].split("(")[0].replace("lik::<unnamed>::", "").replace("lik::", "")
    a = agg.setdefault(name, [0.0, 0])
    a[0] += float(r[v_i].replace(",", ""))
    a[1] += 1
tot = sum(v[0] for v in agg.values())
with open(os.path.join(dst, "launch_shares.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    f.write("command: python bench.py (the default bench run: 3 warm-up + 3 timed steps of C4)\n")
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        f.write(f"{k[:60]:60s} launches={n:5d} total_ms={t/1e6:10.3f} share={t/tot:6.3f}\n")
subprocess.run(["cp", os.path.join(src, "launches.csv"), os.path.join(dst, "launches.csv")])

def raw(rep):
    r = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                   capture_output=True, text=True).stdout)))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}

for kern in ("chol", "build"):
    rep = os.path.join(src, kern + ".ncu-rep")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "20"],
                         capture_output=True, text=True).stdout
    open(os.path.join(dst, f"ncu_{kern}_summary.txt"), "w").write(out)
    m = raw(rep)
    def g(name):
        u, v = m[name]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
        return float(v.replace(",", "")) * scale
    if kern == "chol":
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        pts = int(float(m["launch__grid_size"][1]))
        json.dump({"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "points_per_launch": pts, "dram_bytes_per_point": (rd + wr) / pts,
                   "duration_ms_under_ncu": float(m["gpu__time_duration.sum"][1]),
                   "dmma_pipe_pct": g("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
                   "dmma_pipe_metric": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active (same capture)",
                   "source": f"ncu --set full capture of chol_fused_kernel, profiles/{rnd}/ncu_chol_summary.txt"},
                  open(os.path.join(ROOT, "profiles", "chol_traffic.json"), "w"), indent=1)
print(open(os.path.join(dst, "launch_shares.txt")).read())
print(open(os.path.join(ROOT, "profiles", "chol_traffic.json")).read())
