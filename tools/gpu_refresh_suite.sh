# Second half of tools/gpu_refresh.sh: GPU suite, reference arm, the 8-rank share-gpu line, sweeps.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "reference rc=$?"
python bench.py --gpus 8 --share-gpu --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_share8.log 2>&1; echo "share8 rc=$?"
python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
for k in 1 2 3 4 5 6 7 8 9 10; do echo "a-k$k $(python tools/quick_time.py a-k$k 5 | tail -1)"; done > gpurun_out/problemA.log
for k in 1 2 3 4 5 6 7 8 9 10; do echo "tg-k$k $(python tools/quick_time.py tg-k$k 3 | tail -1)"; done > gpurun_out/tg.log
bash tools/geo_sweep.sh > gpurun_out/geo.log 2>&1
echo done
