#!/usr/bin/env bash
# Quick GPU iteration: parity tests (filter $1), pass microbench, bench line.
set -u
OUT=gpurun_out/${2:-quick}
mkdir -p "$OUT"
timeout 600 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > "$OUT/pytest.log" 2>&1; echo "pytest $?" >> "$OUT/status"
tail -2 "$OUT/pytest.log"
timeout 300 python tools/bench_pass.py > "$OUT/bench_pass.txt" 2>&1; cat "$OUT/bench_pass.txt"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench $?" >> "$OUT/status"
python - "$OUT/bench.json" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.4g  ms %.3f  e2e %.4g  kernel_ms %s  frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, d["roofline"]["frac"]))
for s in d.get("secondary", []): print(s["metric"], s["value"])
PY
