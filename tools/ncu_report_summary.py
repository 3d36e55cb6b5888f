"""Summarise ncu --set full reports (.ncu-rep): per kernel the key speed-of-light,
occupancy and issue metrics plus the SASS opcode mix (from the source page).

    python tools/ncu_report_summary.py report.ncu-rep [...] > profiles/round1/ncu_full_X.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(paths):
    for path in paths:
        print(f"### {path}")
        rows = list(csv.reader(io.StringIO(run([path, "--page", "details", "--csv"]))))
        if not rows:
            continue
        h = rows[0]
        cur = None
        for r in rows[1:]:
            d = dict(zip(h, r))
            k = (d["ID"], d["Kernel Name"][:90])
            if k != cur:
                print(f"== [{k[0]}] {k[1]}")
                cur = k
            if d["Metric Name"] in KEYS:
                print(f"    {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
        # opcode mix per kernel (source page, SASS)
        src = run([path, "--page", "source", "--csv", "--print-source", "sass"])
        kern, ops = None, None
        mixes = []
        for r in csv.reader(io.StringIO(src)):
            if r and r[0] == "Kernel Name":
                ops = collections.Counter()
                mixes.append((r[1][:90], ops))
                continue
            if r and r[0].startswith("0x") and ops is not None:
                op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split(" ")[0]
                ops[op] += int(r[5])
        seen = set()
        for name, ops in mixes:
            if name in seen or not ops:
                continue
            seen.add(name)
            tot = sum(ops.values())
            top = ", ".join(f"{o} {100 * n / tot:.1f}%" for o, n in ops.most_common(8))
            print(f"  SASS mix [{name}] ({tot:.3g} warp-instructions): {top}")


if __name__ == "__main__":
    main(sys.argv[1:])
