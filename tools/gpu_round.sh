#!/usr/bin/env bash
# One GPU-box session: parity tests, bench line, launch lists (+ DRAM bytes) of one
# config-4 certificate and of config-5 cost+gradient. Everything lands in gpurun_out/.
#   gpurun --timeout 1500 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi -q -d CLOCK > "$OUT/clocks_before.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest_gpu exit $?" | tee -a "$OUT/status.txt"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" | tee -a "$OUT/status.txt"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file "$OUT/launches_cert512.csv" \
  python tools/profile_cert.py --n 512 > "$OUT/ncu_cert.log" 2>&1
echo "ncu cert exit $?" | tee -a "$OUT/status.txt"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file "$OUT/launches_costgrad256.csv" \
  python tools/profile_cert.py --costgrad --reps 2 > "$OUT/ncu_cg.log" 2>&1
echo "ncu costgrad exit $?" | tee -a "$OUT/status.txt"
tail -3 "$OUT/pytest_gpu.log"
