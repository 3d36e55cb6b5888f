#!/usr/bin/env bash
# cost+grad (config 5) evals/s and kernel split per env setting (';'-separated VARIANTS)
set -u
IFS=';' read -ra VS <<< "${VARIANTS:-}"
[ ${#VS[@]} -eq 0 ] && VS=("")
for V in "${VS[@]}"; do
  env $V timeout 300 python - <<'PY'
import os, sys, time
sys.path.insert(0, ".")
import bench
class A: cg_steps = 40
r = bench.costgrad_workload(A, 0)
print(os.environ.get("SFW3D_CHUNK32", "-"), "%.1f evals/s" % r["value"], {k: round(v, 4) for k, v in r["kernel_ms"].items()})
PY
done
