set -x
timeout 900 python -m pytest tests/test_gpu_next1.py tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_next1.log 2>&1; echo "next1 rc=$?"
tail -15 gpurun_out/pytest_next1.log
python bench.py --workload a-k7 --steps 20 --warmup 3 --no-e2e --cpu-seconds 10 > gpurun_out/bench_a7.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_a7.log
for k in 1 2 3 4 5 6 8 9 10; do PYTHONPATH=. timeout 300 python tools/quick_time.py a-k$k 5 2>&1 | tail -1; done
