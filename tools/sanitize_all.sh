#!/bin/bash
# compute-sanitizer over the product kernels (tools/sanitize_case.py small / train) and a
# 2-rank shared-GPU bench run; outputs under gpurun_out/san_final/.
cd "$(dirname "$0")/.."
D=gpurun_out/san_final; mkdir -p $D
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py small > $D/small_$tool.txt 2>&1; tail -3 $D/small_$tool.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py train > $D/train_memcheck.txt 2>&1; tail -3 $D/train_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py train > $D/train_racecheck.txt 2>&1; tail -3 $D/train_racecheck.txt
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_case.py small > $D/small_initcheck.txt 2>&1; tail -3 $D/small_initcheck.txt
ODGS_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_2ranks.jsonl 2> $D/bench_2ranks.err; tail -2 $D/bench_2ranks.err; tail -c 300 $D/bench_2ranks.jsonl
