#!/usr/bin/env bash
# Baseline-size parity tests + full bench (parity block) on one box.
set -u
OUT=gpurun_out/${1:-parity}
mkdir -p "$OUT"
free -g > "$OUT/mem.txt"; nproc >> "$OUT/mem.txt"
timeout 1200 python -m pytest tests/test_gpu_baseline_sizes.py -x -q -s > "$OUT/pytest_bs.log" 2>&1; echo "pytest_bs $?" >> "$OUT/status"
tail -5 "$OUT/pytest_bs.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench $?" >> "$OUT/status"
python - "$OUT/bench.json" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.4g ms %.3f e2e %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"]))
print("cpu", d["cpu_baseline"]); print("parity", d["parity"])
PY
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref $?" >> "$OUT/status"
cat "$OUT/bench_ref.json"
