#!/usr/bin/env bash
# GPU test subset (pytest -k filter $1) with timings into gpurun_out/$2.
set -u
OUT=gpurun_out/${2:-tests}
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -q -s --durations=15 ${1:+-k "$1"} > "$OUT/pytest.log" 2>&1; echo "pytest $?" >> "$OUT/status"
tail -25 "$OUT/pytest.log"
