set -u
mkdir -p gpurun_out/narrow
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_ --launch-skip 0 --launch-count 3 \
  -o gpurun_out/narrow/passes python tools/bench_pass.py > gpurun_out/narrow/ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mix_ring --launch-count 1 \
  -o gpurun_out/narrow/mix python tools/profile_cert.py --n 512 > gpurun_out/narrow/ncu_mix.log 2>&1
echo done
