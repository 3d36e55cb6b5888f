set -u
mkdir -p gpurun_out/pass
python tools/bench_pass.py > gpurun_out/pass/bench_pass.txt 2>&1
# one capture per kernel family: wide (89-tap) z and tile passes, narrow (15-tap)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_ --launch-skip 36 --launch-count 6 \
  -o gpurun_out/pass/passes python tools/bench_pass.py > gpurun_out/pass/ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/pass/ncu.log
