"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import re
import sys


def main(path, top=10):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for row in csv.DictReader(lines):
        if row.get("Metric Name") == "gpu__time_duration.sum":
            key = re.sub(r"\(.*", "", row["Kernel Name"])[:70]
            tot[key] += float(row["Metric Value"])
            cnt[key] += 1
    T = sum(tot.values())
    print(f"{path}: total {T / 1e6:.3f} ms over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"  {100 * v / T:6.2f}% {v / 1e6:9.3f} ms {cnt[k]:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
