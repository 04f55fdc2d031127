"""Average the steady-state ncu captures of tools/traffic.sh into
profiles/traffic.json: DRAM bytes (read + write), instructions and duration
per launch at 8K, with the algorithmic bytes and the ratio traffic / alg."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
W, H = 7680, 4320
ALG = {"sr": W * H + (W - 4) * (H - 4) * 24, "sr32": W * H + (W - 4) * (H - 4) * 20,
       "u8": W * H + (W - 4) * (H - 4), "3sr": W * H + (W - 2) * (H - 2) * 16,
       "3u8": W * H + (W - 2) * (H - 2)}


def load(tag):
    rows = list(csv.reader(l for l in open(os.path.join(OUT, f"traffic_{tag}.csv"))
                           if l.startswith('"')))
    h = rows[0]
    by = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = by.setdefault(d["ID"], {"kernel": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6,
                 "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "msecond": 1e-3}.get(unit, 1)
        k[d["Metric Name"]] = v * scale
    return list(by.values())


res = {}
for tag in ALG:
    ls = load(tag)[1:]  # the first captured launch still sees the warm-up's dirty lines start
    n = len(ls)
    rd = sum(l["dram__bytes_read.sum"] for l in ls) / n
    wr = sum(l["dram__bytes_write.sum"] for l in ls) / n
    inst = sum(l["smsp__inst_executed.sum"] for l in ls) / n
    cyc = sum(l["sm__cycles_elapsed.avg"] for l in ls) / n
    us = sum(l["gpu__time_duration.sum"] for l in ls) / n * 1e6
    key = {"sr": "8k/sr", "sr32": "8k/sr32", "u8": "8k/u8", "3sr": "8k/sobel3_sr", "3u8": "8k/sobel3_u8"}[tag]
    res[key] = {"traffic": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                "alg_bytes": ALG[tag], "ratio": (rd + wr) / ALG[tag], "launches": n,
                "inst_per_launch": int(inst), "sm_cycles": cyc, "us_under_ncu": us,
                "issue_frac": inst / (4 * 148 * cyc), "kernel": ls[0]["kernel"]}
res["_source"] = ("ncu --cache-control none --clock-control none, 8 back-to-back launches of "
                  "tools/sweep.py after 5 warm-up ones (tools/traffic.sh), the first captured one "
                  "dropped, the rest averaged (tools/traffic.py): L2 keeps its state between "
                  "launches, so each launch pays the write-back of the previous one's dirty lines "
                  "= steady state.  issue_frac = smsp__inst_executed / (4 SMSPs x 148 SMs x "
                  "sm__cycles_elapsed).  8k/u8 and 8k/sobel3_u8 read less than the algorithmic "
                  "bytes: their 33 MB output plane stays in the 126 MB L2 across the loop "
                  "(the same plane is rewritten each launch), only the rotated inputs come "
                  "from DRAM.")
json.dump(res, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
for k, v in res.items():
    if not k.startswith("_"):
        print(f"{k:16s} traffic {v['traffic']/1e6:7.1f} MB alg {v['alg_bytes']/1e6:7.1f} MB "
              f"ratio {v['ratio']:.3f} inst {v['inst_per_launch']/1e6:5.1f} M "
              f"issue {v['issue_frac']:.3f} {v['us_under_ncu']:.1f} us")
