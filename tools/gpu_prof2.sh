# bench line + launch list + full captures of the fast kernel at k = 7 (C3), 3 and 5 (C4)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 3 -c 1 -o gpurun_out/cell_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
for k in 3 5; do
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 2 -c 1 -o gpurun_out/c4k${k}_full python tools/quick_time.py c4-k$k 2 > gpurun_out/ncu_k$k.log 2>&1; echo "ncu k$k rc=$?"
done
