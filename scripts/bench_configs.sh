#!/bin/bash
# Every BASELINE config through bench.py (contract line: kernel-only value,
# e2e pinned + pageable, roofline, cpu_baseline) and its reference arm, one
# JSON line each, into gpurun_out/configs/.  On the GPU box:
#   gpurun -- bash scripts/bench_configs.sh [tag]
set -u
tag=${1:-r2}
out=gpurun_out/configs
mkdir -p $out
G=$((1 << 30))
run() { # name, args...
    local name=$1; shift
    timeout 1200 python bench.py --steps 10 --warmup 3 "$@" > $out/${tag}_$name.json 2> $out/${tag}_$name.err
    timeout 900 python bench.py --impl reference --steps 2 --warmup 1 "$@" > $out/${tag}_${name}_ref.json 2>> $out/${tag}_$name.err
    echo "$name: $(python scripts/summarize_bench.py $out/${tag}_$name.json $out/${tag}_${name}_ref.json)"
}
for c in ${CONFIGS:-c1 c2 c3 c4:2 c4:4 c4:20 c4:64 c4:128 c4:256 c5:1000 c5:10000 c5:100000 c5:1000000}; do
    name=${c/:/_}
    case $c in
        c1) run $name --config c1 --bytes-per-gpu $((16 << 20)) ;;
        c2) run $name --config c2 --bytes-per-gpu $G ;;
        c3) run $name --config c3 ;;
        c4:*) run $name --config c4 --sigma ${c#c4:} --bytes-per-gpu $G ;;
        c5:*) run $name --config c5 --count ${c#c5:} ;;
    esac
done | tee $out/${tag}_summary.txt
