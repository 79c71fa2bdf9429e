"""Summarise an ncu report: SOL, occupancy, stall reasons, SASS opcode mix.

  python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, rows = raw[0], raw[1], raw[2:]
for row in rows:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "?")[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
            "smsp__inst_executed.sum", "smsp__inst_executed_pipe_fp64.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_bytes.sum"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>14s} {u.get(k, '')}")
    st = {k: float(d[k]) for k in hdr if re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+", k)
          and not k.endswith("not_issued") and d[k] not in ("", "0")}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1]} {v / tot * 100:.0f}%"
                                 for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(src) > 2:
    h = src[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    op = collections.Counter()
    tot = 0
    for r in src[2:]:
        if len(r) <= ia:
            continue
        try:
            n = int(r[ia] or 0)
        except ValueError:   # the header row repeats per kernel in multi-kernel reports
            continue
        tot += n
        toks = r[isrc].split()
        if not toks:
            continue
        o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op[o.split(".")[0]] += n
    print(f"  warp instructions: {tot:.3e}")
    print("  mix:", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in op.most_common(14)))
