set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kern.log 2>&1; echo "kern rc=$?"
tail -5 gpurun_out/pytest_kern.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['e2e'])"
