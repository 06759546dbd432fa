export PYTHONPATH=$PWD
for k in 1 3 5 7; do python tools/quick_time.py tg-k$k 5 2>&1 | tail -1; done
python bench.py --workload tg-k5 --steps 10 --warmup 3 --no-e2e --cpu-seconds 8 > gpurun_out/bench_tg5.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/bench_tg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['parity'], d['kernel_info'], d['roofline']['kernel'])"
