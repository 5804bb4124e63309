#!/bin/bash
# Measurement pass for one round (on the GPU box: gpurun -- bash scripts/profile_round.sh <tag>).
# Writes gpurun_out/<tag>/:
#   bench.json, bench_ref.json      the contract line (c3) and its reference arm
#   launches.csv                    ncu launch list (gpu__time_duration) of a short bench run
#   ncu_<kernel>.ncu-rep + _details.txt  ncu --set full of the dominant kernels:
#                                   c3 filter + walking pass, c2 pack + direct-index kernel,
#                                   c5 1M single+L2 filter pass
#   probe_configs.jsonl             every config state at 1 GiB with full-array parity
#                                   (memcmp + SHA-256) against the compiled reference
set -u
tag=${1:-r2}
out=gpurun_out/$tag
mkdir -p $out
G=1073741824
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2>> $out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > /dev/null 2>> $out/bench.err
# ncu --set full of one kernel; keeps text exports (details page, raw
# counters, per-source-line instruction and stall shares) and drops the
# report itself (gpurun copies back at most 64 MiB)
prof() { # name, kernel regex, launches to capture, mangled kernel name for the line split, bench args...
    local name=$1 k=$2 c=$3 mangled=$4; shift 4
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 3 -c $c \
        -o /tmp/ncu_$name python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 "$@" \
        > /dev/null 2>> $out/bench.err
    ncu -i /tmp/ncu_$name.ncu-rep --page details > $out/ncu_${name}_details.txt 2>/dev/null
    ncu -i /tmp/ncu_$name.ncu-rep --page raw --csv > $out/ncu_${name}_raw.csv 2>/dev/null
    python scripts/ncu_lines.py /tmp/ncu_$name.ncu-rep paper_1704_02272_b200/build/engine.o "$mangled" 40 \
        > $out/ncu_${name}_lines.txt 2>&1
    rm -f /tmp/ncu_$name.ncu-rep
}
prof c3_filter pfac_pair_filter_kernel 1 _ZN3hfb3gpu23pfac_pair_filter_kernelILb0EEEvNS0_10FilterArgsE --bytes-per-gpu $G
prof c3_walk 'pfac_scan_kernel' 1 _ZN3hfb3gpu16pfac_scan_kernelILb1ELb1ELi3ELb0ELb1EEEvNS0_8ScanArgsE --bytes-per-gpu $G
prof c2_dna 'pfac_dna_kernel' 1 _ZN3hfb3gpu15pfac_dna_kernelILj32EEEvNS0_8ScanArgsE --config c2 --bytes-per-gpu $G
prof c2_pack 'pfac_pack_dna' 1 _ZN3hfb3gpu20pfac_pack_dna_kernelILb1EEEvPKhmPKtjPjS6_m --config c2 --bytes-per-gpu $G
prof c5m_l2 pfac_l2_filter_kernel 1 _ZN3hfb3gpu21pfac_l2_filter_kernelILi3EEEvNS0_10FilterArgsE --config c5 --count 1000000 --bytes-per-gpu $G
if [ "${PROBE:-1}" = 1 ]; then
timeout 2400 python scripts/probe.py --check --full-check --iters 5 \
    --configs ${PROBE_CONFIGS:-c1,c2,c3,c4:2,c4:4,c4:20,c4:64,c4:128,c4:256,c5:1000,c5:10000,c5:100000,c5:1000000} \
    > $out/probe_configs.jsonl 2>> $out/bench.err
fi
echo done
