#!/usr/bin/env bash
# Config-4 certificate bench line (and the pass microbenchmark) per env setting.
#   VARIANTS='A=1;A=1 B=2;' bash tools/env_scan.sh tag   (';'-separated, empty = default)
set -u
OUT=gpurun_out/${1:-scan}; mkdir -p $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-}"
[ ${#VS[@]} -eq 0 ] && VS=("")
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  echo "== [$V]"
  env $V timeout 300 python tools/bench_pass.py 2>&1 | tail -2
  env $V timeout 300 python bench.py --no-secondary --no-cpu-baseline > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  python - $OUT/bench_$i.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.4g ms %.3f refined %s best %s kernel_ms %s" % (d["value"], d["ms_per_step"], d["refined_voxels"], d["argmax"], {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}))
PY
done
