#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck (+ synccheck) over a GPU test subset:
# the certificate (fold / mix / collect / refine kernels incl. the slab path),
# the passes, cost + gradient, LASSO. Logs into gpurun_out/$1.
set -u
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
SUB="tests/test_gpu_parity.py tests/test_gpu_certificate.py::test_eta_f32_basis_vs_oracle tests/test_gpu_certificate.py::test_signed_members_refined_maxima tests/test_gpu_certificate.py::test_table_fits tests/test_gpu_passes.py::test_psf_passes_vs_fft"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest $SUB -x -q -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool exit $?" | tee -a $OUT/status
  grep -E "ERROR SUMMARY|passed|failed" $OUT/$tool.log | tail -3
done
