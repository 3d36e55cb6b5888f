# ncu --set full of the config-5 cost + gradient kernels (render, atom sums)
set -u
OUT=gpurun_out/${1:-cg}
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"render|atom_sums" --launch-skip 4 --launch-count 2 \
  -o $OUT/cg python tools/profile_cert.py --costgrad --reps 4 > $OUT/ncu.log 2>&1
echo "ncu $?"
