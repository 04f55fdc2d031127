"""SURVEY 8(d) evidence from an .ncu-rep (--set full): DRAM bytes and
throughput, L2 hit rate, shared-memory vs shuffle traffic (instruction
counts from the SASS source page), TMA and global-memory instruction
counts, pipe utilisation.  usage: python tools/ncu_evidence.py <rep> [...]"""
import csv
import io
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "kernel time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of ncu peak)"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("smsp__inst_executed.sum", "warp-instructions"),
    ("smsp__sass_inst_executed_op_global_ld.sum", "LDG (global loads)"),
    ("smsp__sass_inst_executed_op_global_st.sum", "STG (global stores)"),
    ("smsp__sass_inst_executed_op_tma_ld.sum", "TMA bulk loads"),
    ("smsp__sass_inst_executed_op_tma_st.sum", "TMA stores"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "LDS (shared loads)"),
    ("smsp__sass_inst_executed_op_shared_st.sum", "STS (shared stores)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed", "XU pipe (MUFU) %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def page(rep, p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    raw = page(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    print(f"== {d.get('Kernel Name')}")
    for key, name in RAW:
        if key in d:
            print(f"  {name:34s} {d[key]} {u.get(key, '')}  ({key})")
    src = page(rep, "source", ("--print-source", "sass"))
    h = src[1]
    isrc, iexe = h.index("Source"), h.index("Instructions Executed")
    counts = {}
    for r in src[2:]:
        op = r[isrc].split()
        if not op:
            continue
        mn = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        mn = mn.split(".")[0]
        try:
            counts[mn] = counts.get(mn, 0) + int(float(r[iexe] or 0))
        except ValueError:
            pass
    tot = sum(counts.values()) or 1
    for mn in ("SHFL", "LDS", "STS", "LDG", "STG", "UBLKCP", "UTMASTG", "PRMT", "IMAD", "IADD3",
               "FFMA2", "FADD2", "FMUL2", "MUFU", "DFMA", "DMUL"):
        if counts.get(mn):
            print(f"  SASS {mn:8s} executed {counts[mn]:>12d} warp-instr ({counts[mn] / tot * 100:5.1f}%)")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
