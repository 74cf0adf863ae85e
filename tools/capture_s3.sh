#!/bin/bash
# Session-3 evidence: compute-sanitizer over the small / bigsort cases (gpurun_out/san_s3/), then
# tools/final_capture.sh.
cd "$(dirname "$0")/.."
D=gpurun_out/san_s3; mkdir -p $D
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py small > $D/small_$tool.txt 2>&1; tail -1 $D/small_$tool.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py bigsort > $D/bigsort_memcheck.txt 2>&1; tail -1 $D/bigsort_memcheck.txt
bash tools/final_capture.sh
