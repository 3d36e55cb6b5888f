"""Summarise an ncu report (details page) into a compact per-kernel table."""
import csv
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Theoretical Occupancy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "FP32 Peak", "Warp Cycles Per Issued Instruction")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    cur = None
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        key = (d["ID"], d["Kernel Name"][:60])
        if key != cur:
            print("==", *key)
            cur = key
        if d["Metric Name"] in WANT:
            print(f"    {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")


if __name__ == "__main__":
    main(sys.argv[1])
