#!/usr/bin/env bash
# Full solves (configs 2, 3) at the default basis settings and at $OLD.
set -u
OUT=gpurun_out/${1:-solves}; mkdir -p $OUT
for c in 2 3; do
  echo "cfg$c default: $(timeout 600 python tools/run_solve.py --config $c 2>$OUT/cfg${c}_new.err | tail -1)"
  [ -n "${OLD:-}" ] && echo "cfg$c [$OLD]: $(env $OLD timeout 600 python tools/run_solve.py --config $c 2>$OUT/cfg${c}_old.err | tail -1)"
done
