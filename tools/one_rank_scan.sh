#!/usr/bin/env bash
# Per-rank certificate time of the x-slab layout for W = 2, 4, 8, one rank at a
# time on this GPU (no process group): the max over ranks predicts the W-GPU
# step (ranks exchange only the argmax records).
set -u
OUT=gpurun_out/onerank; mkdir -p $OUT
for W in ${WS:-2 4 8}; do
  for R in $(seq 0 $((W - 1))); do
    [ "$R" -gt 1 ] && [ "${ALL:-0}" = 0 ] && break   # slabs are equal-sized: ranks 0-1 suffice
    timeout 600 python bench.py --one-rank $R/$W --no-secondary --no-cpu-baseline --steps 5 > $OUT/w${W}_r${R}.json 2> $OUT/w${W}_r${R}.err
    python - $OUT/w${W}_r${R}.json <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(d["one_rank"], "ms/step %.3f" % d["ms_per_step"], "halo", d["config"]["parallelism"][:60], "best", d["argmax"])
PY
  done
done
