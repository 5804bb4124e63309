#!/bin/bash
# compute-sanitizer over every kernel form (scripts/sanitize_cases.py), one
# process per (tool, case); logs under gpurun_out/sanitize/.  Run on the GPU
# box: gpurun -- bash scripts/sanitize.sh
set -u
out=gpurun_out/sanitize
mkdir -p $out
cases="${CASES:-fused_pair fused_single fused_dna two_pass_pair two_pass_pair_l2 two_pass_l2 symbol streamed session}"
for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
    for c in $cases; do
        timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
            python scripts/sanitize_cases.py $c > $out/${tool}_$c.log 2>&1
        echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok$|MISMATCH' $out/${tool}_$c.log | tr '\n' ' ')"
    done
done | tee $out/summary.txt
