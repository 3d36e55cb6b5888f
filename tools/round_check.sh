#!/usr/bin/env bash
# Full round check on one box: GPU tests, smoke, default bench line, reference arm.
set -u
OUT=gpurun_out/${1:-round}
mkdir -p $OUT
nvidia-smi -q -d CLOCK > $OUT/clocks_before.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu $?" | tee -a $OUT/status
tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?" | tee -a $OUT/status
tail -1 $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" | tee -a $OUT/status
timeout 1200 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref $?" | tee -a $OUT/status
python - $OUT/bench.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.4g ms %.3f e2e %.4g frac %.3f launches %s" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d.get("gpu_launches")))
print("parity", d["parity"]); print("cpu", d["cpu_baseline"]["value"])
for s in d["secondary"]: print(s["metric"], round(s["value"],4), s.get("cpu_baseline",{}).get("value") if s.get("cpu_baseline") else "")
PY
