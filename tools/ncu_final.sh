#!/usr/bin/env bash
# ncu --set full captures of the config-4 certificate's top kernels (one launch each).
set -u
OUT=gpurun_out/final; mkdir -p $OUT
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:pass_tile2_kernel --launch-skip 4 --launch-count 1 -o $OUT/tile2 python tools/profile_cert.py --n 512 > $OUT/tile2.log 2>&1
timeout 600 $N -k regex:pass_z2_kernel --launch-skip 2 --launch-count 1 -o $OUT/z2 python tools/profile_cert.py --n 512 > $OUT/z2.log 2>&1
timeout 600 $N -k regex:mix_ring2 --launch-count 1 -o $OUT/mix python tools/profile_cert.py --n 512 > $OUT/mix.log 2>&1
timeout 600 $N -k regex:"atom_sums_kernel|render_kernel" --launch-skip 2 --launch-count 2 -o $OUT/cg python tools/profile_cert.py --costgrad --reps 2 > $OUT/cg.log 2>&1
ls $OUT
