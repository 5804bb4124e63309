#!/bin/bash
# Measurement pass for one round (run on the GPU box through gpurun):
#   scripts/profile_round.sh <tag>
# writes gpurun_out/{bench,bench_ref}_<tag>.json, launches_<tag>.csv and
# ncu --set full captures of both scan kernels (c3, 1 GiB) as .ncu-rep + .txt.
set -u
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_$tag.json 2>> $out/bench_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_$tag.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
    > /dev/null 2>> $out/bench_$tag.err
for k in pfac_pair_filter_kernel pfac_scan_kernel; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 \
        -o $out/ncu_${tag}_$k python bench.py --bytes-per-gpu 1073741824 --steps 2 --warmup 1 \
        --no-cpu-baseline --e2e-steps 1 > /dev/null 2>> $out/bench_$tag.err
    ncu -i $out/ncu_${tag}_$k.ncu-rep --page details > $out/ncu_${tag}_${k}_details.txt 2>/dev/null
done
echo done
