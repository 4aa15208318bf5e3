"""Summarise an ncu report: key metrics, stall reasons and the SASS opcode mix."""
import csv, io, subprocess, sys
from collections import Counter

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__cycles_elapsed.avg",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

def main(rep, sass=True):
    h, u, rows = raw(rep)
    for r in rows:
        print("kernel:", r[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k:60s} {r[h.index(k)]:>16s} {u[h.index(k)]}")
        st = [(h[i], float(r[i].replace(",", "") or 0)) for i in range(len(h))
              if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
        tot = sum(v for _, v in st) or 1
        print("  stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*v/tot:.0f}%"
                                      for n, v in sorted(st, key=lambda x: -x[1])[:8]))
    if sass:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hh = rows[1]
        isrc, iex = hh.index("Source"), hh.index("Instructions Executed")
        c = Counter()
        tot = 0
        for r in rows[2:]:
            if len(r) < len(hh):
                continue
            ex = float(r[iex] or 0)
            toks = r[isrc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            c[op.split(".")[0]] += ex
            tot += ex
        print(f"  SASS executed {tot:.3e}: " + ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in c.most_common(14)))

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
