#!/usr/bin/env bash
# Round-2 evidence: ncu launch lists (time + DRAM bytes per launch, base units)
# of one config-4 certificate and config-5 cost + gradient, and --set full
# captures of the top kernels. Everything under gpurun_out/$1.
set -u
OUT=gpurun_out/${1:-ncu2}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --print-units base --csv --log-file $OUT/launches_cert512.csv \
  python tools/profile_cert.py --n 512 --reps 2 > $OUT/l_cert.log 2>&1; echo "launch cert $?"
timeout 900 ncu --metrics $M --clock-control none --print-units base --csv --log-file $OUT/launches_costgrad256.csv \
  python tools/profile_cert.py --costgrad --reps 3 > $OUT/l_cg.log 2>&1; echo "launch cg $?"
N="ncu --set full --import-source on --clock-control none"
timeout 900 $N -k regex:pass_tile2x2_kernel --launch-skip 2 --launch-count 1 -o $OUT/tile2x2 python tools/profile_cert.py --n 512 > $OUT/f1.log 2>&1; echo "full tile2x2 $?"
timeout 900 $N -k regex:pass_z2_kernel --launch-skip 0 --launch-count 1 -o $OUT/z2 python tools/profile_cert.py --n 512 > $OUT/f2.log 2>&1; echo "full z2 $?"
timeout 900 $N -k regex:mix_ring2 --launch-count 1 -o $OUT/mix python tools/profile_cert.py --n 512 > $OUT/f3.log 2>&1; echo "full mix $?"
timeout 900 $N -k regex:"atom_sums_f32|render_f32|pass_tile2_kernel" --launch-skip 4 --launch-count 4 -o $OUT/cg python tools/profile_cert.py --costgrad --reps 3 > $OUT/f4.log 2>&1; echo "full cg $?"
ls -la $OUT
