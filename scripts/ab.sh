# usage: ab.sh "configs" states variant... (variant = name[:ENV=VAL])
C=$1; S=$2; shift 2
for r in 1 2; do for v in "$@"; do n=${v%%:*}; e=""; [ "$n" != "$v" ] && e=${v#*:}; if [ "$n" = cur ]; then L=$PWD/paper_1704_02272_b200/libhepfac.so; else L=$PWD/paper_1704_02272_b200/libhepfac_$n.so; fi
env $e HEPFAC_LIB=$L timeout 300 python scripts/probe.py --configs $C --states $S > gpurun_out/ab.jsonl 2>/dev/null
echo "$v: $(python -c "
import json
print(' '.join(f\"{d['config']}/{d['state'][:3]}={d['GBps']}\" for d in map(json.loads, open('gpurun_out/ab.jsonl'))))")"; done; done
