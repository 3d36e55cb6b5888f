set -u
mkdir -p gpurun_out/cg
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"render_kernel|atom_sums_kernel|sumsq" --launch-skip 3 --launch-count 4 \
  -o gpurun_out/cg/cg python tools/profile_cert.py --costgrad --reps 2 > gpurun_out/cg/ncu.log 2>&1
echo done
