#!/usr/bin/env bash
# Scan SFW3D_BASIS_LOOSE on the config-4 certificate (bench line per value)
# and run the certificate parity tests at one loose value.
set -u
OUT=gpurun_out/loose; mkdir -p $OUT
SFW3D_BASIS_LOOSE=${TESTL:-1.5e-6} timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for L in ${LIST:-0 1e-7 3e-7 1.5e-6}; do
  SFW3D_BASIS_LOOSE=$L timeout 300 python bench.py --no-secondary --no-cpu-baseline > $OUT/bench_$L.json 2> $OUT/bench_$L.err
  python - $OUT/bench_$L.json $L <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], "value %.4g ms %.3f refined %s best %s kernel_ms %s" % (d["value"], d["ms_per_step"], d["refined_voxels"], d["argmax"], {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}))
PY
done
