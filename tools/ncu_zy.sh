set -u
OUT=gpurun_out/${1:-ncuzy}
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pass_zy_kernel" --launch-skip 2 --launch-count 1 \
  -o $OUT/zy python tools/bench_pass.py > $OUT/ncu.log 2>&1
echo "ncu $?"
