# ncu --set full of the config-4 certificate's pass kernels (one narrow z, one narrow strided,
# one wide z, one wide strided) and the mix
set -u
OUT=gpurun_out/${1:-ncupass}
mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"pass_z2_kernel|pass_tile2_kernel|mix_ring2" \
  --launch-skip 0 --launch-count 9 -o $OUT/pass python tools/profile_cert.py --n 512 --reps 1 > $OUT/ncu.log 2>&1
echo "ncu $?"
