"""Summarise an ncu report: key SOL/occupancy/memory metrics and the SASS opcode mix per kernel."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

KEYS = ("Duration", "Elapsed Cycles", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "No Eligible", "Eligible Warps Per Scheduler")


def run(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(rep, opmix=True):
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seen = {}
    for r in rows[1:]:
        k = re.sub(r"\(.*", "", r[ki]).replace("void <unnamed>::", "")
        if r[mi] in KEYS:
            seen.setdefault(k, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    for k, d in seen.items():
        print(f"== {k}")
        for key in KEYS:
            if key in d:
                print(f"   {key:38s} {d[key]}")
    raw = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv", "--metrics",
                                           "dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,"
                                           "lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct"]))))
    if raw:
        hh = raw[0]
        for r in raw[2:]:
            d = dict(zip(hh, r))
            k = re.sub(r"\(.*", "", d.get("Kernel Name", "")).replace("void <unnamed>::", "")
            print(f"-- {k}: dram read {d.get('dram__bytes_read.sum')} write {d.get('dram__bytes_write.sum')} "
                  f"inst {d.get('smsp__inst_executed.sum')} L2 hit {d.get('lts__t_sector_hit_rate.pct')} "
                  f"L1 hit {d.get('l1tex__t_sector_hit_rate.pct')}  (units row: {raw[1][hh.index('dram__bytes_read.sum')] if 'dram__bytes_read.sum' in hh else ''})")
    if not opmix:
        return
    for kern in ("march", "build"):
        src = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"]))))
        if len(src) < 3:
            continue
        h = src[1]
        si, ii, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        op, st, tot, totw = Counter(), Counter(), 0, 0
        for r in src[2:]:
            if len(r) != len(h):
                continue
            try:
                n, w = int(r[ii] or 0), int(r[ws] or 0)
            except ValueError:
                continue
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si])
            o = m.group(2) if m else "?"
            op[o] += n
            st[o] += w
            tot += n
            totw += w
        print(f"== opcode mix {kern}: {tot} warp-inst, {totw} stall samples")
        for o, n in op.most_common(24):
            print(f"   {o:10s} {100 * n / tot:5.1f}% inst {100 * st[o] / max(totw, 1):5.1f}% stall")


if __name__ == "__main__":
    main(sys.argv[1], opmix="--no-opmix" not in sys.argv)
