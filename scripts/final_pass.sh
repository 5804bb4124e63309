#!/bin/bash
# The round's final measurement pass in one gpurun call:
#   profile_round.sh (contract line, reference arm, launch list, ncu exports,
#   every config with full-array parity), the per-config contract lines
#   (bench_configs.sh) and the sanitizers.  Output: gpurun_out/<tag>/,
#   gpurun_out/configs/<tag>_*, gpurun_out/sanitize/.
set -u
tag=${1:-r2final}
bash scripts/profile_round.sh $tag > /dev/null 2>&1
bash scripts/bench_configs.sh $tag > /dev/null 2>&1
bash scripts/sanitize.sh > /dev/null 2>&1
python scripts/summarize_bench.py gpurun_out/$tag/bench.json gpurun_out/$tag/bench_ref.json
cat gpurun_out/configs/${tag}_summary.txt gpurun_out/sanitize/summary.txt
