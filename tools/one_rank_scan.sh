#!/usr/bin/env bash
# Per-rank certificate step of a W-rank x-slab layout, each rank run ALONE on
# this GPU (bench.py --one-rank R/W: SoloComm, halos filled locally) — the
# compute side of the multi-GPU projection; NVLink time is added separately.
set -u
OUT=gpurun_out/${1:-onerank}
mkdir -p $OUT
for W in 2 4 8; do
  for R in 0 $((W-1)); do
    timeout 300 python bench.py --one-rank $R/$W --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > $OUT/r${R}_w${W}.json 2> $OUT/r${R}_w${W}.err
    python -c "import json;d=json.load(open('$OUT/r${R}_w${W}.json'));print('W=$W R=$R ms', round(d['ms_per_step'],3), 'halo MiB', round(d.get('halo_mib_received_per_step') or 0,1), 'kernels', {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
  done
done
