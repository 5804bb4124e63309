set -u
bash scripts/sanitize.sh > /dev/null 2>&1
python scripts/_memcpy_bench.py > gpurun_out/memcpy_bench.txt 2>&1
bash scripts/bench_configs.sh r2c > /dev/null 2>&1
cat gpurun_out/sanitize/summary.txt gpurun_out/memcpy_bench.txt gpurun_out/configs/r2c_summary.txt
