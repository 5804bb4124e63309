#!/bin/bash
# Builds kernel variants (compile-time switches in scan_kernel.cuh) as
# paper_1704_02272_b200/libhepfac_<name>.so for A/B runs on the GPU:
#   HEPFAC_LIB=$PWD/paper_1704_02272_b200/libhepfac_<name>.so python scripts/probe.py ...
# usage: scripts/variants.sh name "-DHFB_X=1 -DHFB_Y=2" [name "flags"] ...
set -e
cd "$(dirname "$0")/../paper_1704_02272_b200"
while [ $# -ge 2 ]; do
    make -s -j8 B="build_$1" LIB="libhepfac_$1.so" EXTRA="$2" "libhepfac_$1.so" >/dev/null
    echo "$1: $(grep -E 'Used' build_$1/ptxas.log | awk '{print $5}' | sort -n | tail -1) regs max, spills: $(grep -c 'spill stores' build_$1/ptxas.log) lines, $(grep 'spill' build_$1/ptxas.log | awk '{s+=$5} END {print s+0}') bytes"
    shift 2
done
