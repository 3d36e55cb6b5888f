set -u
mkdir -p gpurun_out/zy
timeout 300 python -m pytest tests/test_gpu_passes.py -x -q 2>&1 | grep -E "assert|Error|passed|failed" | head -5
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_zy --launch-count 1 \
  -o gpurun_out/zy/zy python tools/bench_pass.py > gpurun_out/zy/ncu.log 2>&1
echo done
