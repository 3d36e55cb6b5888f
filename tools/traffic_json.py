"""DRAM bytes per launch per kernel family from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).

    python tools/traffic_json.py launches_cert512.csv > profiles/round1/traffic_cert512.json
"""
import collections
import csv
import json
import re
import sys

FAMILIES = (("eta_basis", r"pass_(tile|z|tiled|zy)"), ("render", r"render"),
            ("atom_sums", r"atom_sums"), ("eta_mix", r"mix_argmax_kernel<[^>]*, 0>|mix_ring2?_kernel"),
            ("eta_direct", r"eta_(fold|direct|sym)_kernel"), ("eta_refine", r"refine_kernel"))


def main(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = collections.defaultdict(dict)
    names = {}
    for row in csv.DictReader(lines):
        per[row["ID"]][row["Metric Name"]] = row["Metric Value"]
        names[row["ID"]] = row["Kernel Name"]
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        for f, pat in FAMILIES:
            if re.search(pat, names[i]):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(m["dram__bytes_read.sum"].replace(",", ""))
                wr = float(m["dram__bytes_write.sum"].replace(",", ""))
                fam[f][0] += 1
                fam[f][1] += rd + wr
                fam[f][2] += float(m["gpu__time_duration.sum"].replace(",", ""))
                break
    out = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none ({path})",
           "families": {f: {"launches": n, "dram_bytes_per_launch": b / n, "ncu_ms_per_launch": t / n / 1e6}
                        for f, (n, b, t) in fam.items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
