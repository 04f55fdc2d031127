"""Summarise an .ncu-rep: key metrics, stall breakdown, top stalled SASS."""
import csv, io, subprocess, sys
rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    print(f"{k:60s} {d.get(k)} {u.get(k, '')}")
if len(sys.argv) > 2:
    src = page("source", ("--print-source", "sass"))
    h = src[1]; data = src[2:]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in cols}
    T = sum(tot.values()) or 1
    print("stalls:", ", ".join(f"{c[6:]} {v/T*100:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    S = sum(float(r[iss] or 0) for r in data) or 1
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:int(sys.argv[2])]:
        reasons = {c[6:]: int(float(r[h.index(c)])) for c in cols if float(r[h.index(c)] or 0) > 0.1 * float(r[iss] or 1)}
        print(f"{r[ia][-5:]} {float(r[iss])/S*100:5.1f}% {r[isrc][:70]:70s} {reasons}")
