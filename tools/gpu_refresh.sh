# Round-end refresh on one B200 (run under gpurun): GPU suite, bench line, launch list,
# ncu --set full captures of the operator kernels, degree / workload sweeps.
# Every ncu command follows a plain run of the same command that exited 0 (B200_PROFILING.md).
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c3b.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 3 -c 1 -o gpurun_out/cell_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu C3 rc=$?"
for w in a-k7 c-k7 tg-k5; do
  python tools/quick_time.py $w 2 > gpurun_out/plain_$w.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"dg_(gen|geo|vb)_kernel" -s 2 -c 1 -o gpurun_out/${w}_full python tools/quick_time.py $w 2 > gpurun_out/ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
