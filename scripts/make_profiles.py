"""Copy the round's ncu evidence into profiles/: launch-list shares, per-kernel
summaries (dram bytes, issue, stalls, SASS mix) and profiles/ncu_traffic.json
(dram read+write bytes per launch of the dominant kernels, read by bench.py)."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

# launch list -> per-kernel totals and shares
rows = list(csv.reader(open(os.path.join(G, f"launches_{R}.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("es::<unnamed>::", "").strip()
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
allns = sum(tot.values())
with open(os.path.join(P, f"{R}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 --warmup 1 --ncu (cold-cache, serialised)\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total_ns':>12s} {'share':>7s}\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"{k[:60]:60s} {cnt[k]:8d} {v:12.0f} {100 * v / allns:6.1f}%\n")

traffic = {}
for tag, kern in [("k2", "k2_replay"), ("k3", "k3_stats"), ("k1", "k1_call"), ("k1h", "k1_harvested"),
                  ("k1clip", "k1_clip")]:
    rep = os.path.join(G, f"prof_{tag}_{R}.ncu-rep")
    if not os.path.exists(rep):
        continue
    s = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep], capture_output=True,
                       text=True).stdout
    open(os.path.join(P, f"{R}_ncu_{tag}.txt"), "w").write(s)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    hh, uu = rr[0], rr[1]
    def val(row, m):
        x = float(row[hh.index(m)].replace(",", ""))
        u = uu[hh.index(m)]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    total = 0.0
    issue = {}
    for row in rr[2:]:
        nm = row[hh.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
        issue[nm] = {"issue_active_pct": float(row[hh.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]
                                                .replace(",", "")),
                     "warp_inst": val(row, "smsp__inst_executed.sum") if "smsp__inst_executed.sum" in hh else None}
    traffic.setdefault("_issue", {}).update(issue)
    for row in rr[2:]:  # one row per captured launch (K1: the four kernels of one call)
        b = val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum")
        name = row[hh.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0].strip()
        name = name.replace("void ", "")
        if tag == "k1":
            traffic[name] = b
        total += b
    traffic[kern] = total
json.dump({**traffic, "_source": f"ncu --set full, {R}, dram__bytes_read.sum + dram__bytes_write.sum per launch"},
          open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(P, f"{R}_launches.txt")).read())
print(traffic)
