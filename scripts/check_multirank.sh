set -u
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --bytes-per-gpu 268435456 --no-cpu-baseline --check > gpurun_out/check2.json 2> gpurun_out/check2.err; echo "rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 3 --steps 3 --warmup 3 --bytes-per-gpu 100000007 --config c2 --trie stage2 --no-cpu-baseline --check > gpurun_out/check3.json 2> gpurun_out/check3.err; echo "rc=$?"
python -c "
import json
for f in ('check2','check3'):
    try:
        d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['check'], d['config']['parallelism'], d['value'], d['e2e']['value'], d['e2e_pageable']['value'])
    except Exception as e: print(f, 'ERR', e); print(open('gpurun_out/'+f+'.err').read()[-3000:])
"
timeout 1200 python -m pytest tests -m gpu -q -k "engine or configs or session or streamed or multi_device" > gpurun_out/gputest_r2f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_r2f.log
