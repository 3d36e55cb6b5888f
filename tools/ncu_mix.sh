set -u
mkdir -p gpurun_out/mix2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mix_ring --launch-count 1 \
  -o gpurun_out/mix2/mix python tools/profile_cert.py --n 512 > gpurun_out/mix2/ncu_mix.log 2>&1
echo done
