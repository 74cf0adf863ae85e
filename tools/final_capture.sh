#!/bin/bash
# Round-end evidence in one GPU call: the GPU test suite, the bench line and the
# reference arm, the ncu launch list of a short bench run, and ncu --set full captures of
# the C3 blend and the C4 backward kernels. Outputs under gpurun_out/final_*.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1
tail -2 gpurun_out/final_gputest.log
python bench.py > gpurun_out/final_bench.jsonl 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 900 --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --train-steps 1 \
    > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_blend_cull -s 20 -c 1 \
    -o gpurun_out/final_c3_blend python tools/profile_c3.py 30 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_bwd_raster_cull|k_fold_records|k_bwd_splat" -c 3 \
    -o gpurun_out/final_c4_bwd python tools/profile_c4_view.py 1 > /dev/null 2>&1
ls -la gpurun_out | grep final
