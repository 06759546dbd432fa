export PYTHONPATH=$PWD; mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --submesh-check > gpurun_out/bench_c3.log 2>&1; echo "bench C3 rc=$?"
for w in c5weak c5strong a-k7 c-k7 tg-k5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --submesh-check > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"
done
