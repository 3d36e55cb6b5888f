#!/usr/bin/env bash
# Round-2 (second half) evidence: launch lists with DRAM bytes of a config-4
# certificate and config-5 cost + gradient at HEAD, and --set full captures of
# the pass tiles, the mix, the single-atom ascent kernel and the ranged residual.
set -u
OUT=gpurun_out/${1:-ncu3}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --print-units base --csv --log-file $OUT/launches_cert512.csv \
  python tools/profile_cert.py --n 512 --reps 2 > $OUT/l_cert.log 2>&1; echo "launch cert $?"
timeout 900 ncu --metrics $M --clock-control none --print-units base --csv --log-file $OUT/launches_costgrad256.csv \
  python tools/profile_cert.py --costgrad --reps 3 > $OUT/l_cg.log 2>&1; echo "launch cg $?"
N="ncu --set full --import-source on --clock-control none"
timeout 900 $N -k regex:pass_tile2x2_kernel --launch-skip 2 --launch-count 1 -o $OUT/tile2x2_narrow python tools/profile_cert.py --n 512 > $OUT/f1.log 2>&1; echo "full tile2x2 narrow $?"
timeout 900 $N -k regex:pass_tile2x2_kernel --launch-skip 20 --launch-count 1 -o $OUT/tile2x2_wide python tools/profile_cert.py --n 512 > $OUT/f1b.log 2>&1; echo "full tile2x2 wide $?"
timeout 900 $N -k regex:pass_z2_kernel --launch-skip 0 --launch-count 1 -o $OUT/z2 python tools/profile_cert.py --n 512 > $OUT/f2.log 2>&1; echo "full z2 $?"
timeout 900 $N -k regex:mix_ring2 --launch-count 1 -o $OUT/mix python tools/profile_cert.py --n 512 > $OUT/f3.log 2>&1; echo "full mix $?"
timeout 900 $N -k regex:refine_sums_kernel --launch-skip 10 --launch-count 2 -o $OUT/refine_sums python tools/refine_probe.py > $OUT/f5.log 2>&1; echo "full refine_sums $?"
timeout 900 $N -k regex:residual_kernel --launch-skip 2 --launch-count 2 -o $OUT/residual python tools/lasso_step_probe.py 100 > $OUT/f6.log 2>&1; echo "full residual $?"
timeout 900 $N -k regex:"atom_sums_f32|render_f32" --launch-skip 2 --launch-count 2 -o $OUT/cg python tools/profile_cert.py --costgrad --reps 3 > $OUT/f4.log 2>&1; echo "full cg $?"
ls -la $OUT
