# First half of tools/gpu_refresh.sh: ncu captures of this build's operator kernels (each after a
# plain run of the same command that exited 0), their summaries, the launch list, the C3 bench line
# and smoke(). Run under gpurun; copy gpurun_out/ncu_full_summary.json to profiles/ afterwards.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 3 -c 1 -o gpurun_out/c3_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu C3 rc=$?"
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c3l.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python bench.py --workload c5weak --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c5w.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 3 -c 1 -o gpurun_out/c5w_full python bench.py --workload c5weak --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c5w.log 2>&1; echo "ncu C5 weak rc=$?"
for w in c4-k8 c4-k10; do
  python tools/quick_time.py $w 2 > gpurun_out/plain_$w.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"dg_cell_kernel" -s 3 -c 1 -o gpurun_out/${w}_full python tools/quick_time.py $w 2 > gpurun_out/ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
for w in a-k7 c-k7 tg-k5; do
  python tools/quick_time.py $w 2 > gpurun_out/plain_$w.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"dg_(gen|geo|vb)_kernel" -s 2 -c 1 -o gpurun_out/${w}_full python tools/quick_time.py $w 2 > gpurun_out/ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
for a in "c3_full C3 268435456" "c5w_full C5-weak-P1 536870912" "c4-k8_full C4-k8 102503232" "c4-k10_full C4-k10 98611128" "a-k7_full A-k7 398688256" "c-k7_full C-k7 398688256" "tg-k5_full TG-k5 401947272"; do
  set -- $a; [ -f gpurun_out/$1.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$1.ncu-rep --name $2 --ndofs $3 --json profiles/ncu_full_summary.json > /dev/null
done
cp profiles/ncu_full_summary.json gpurun_out/ncu_full_summary.json
python bench.py --steps 20 --warmup 5 --submesh-check > gpurun_out/bench_c3.log 2>&1; echo "bench C3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for w in c5weak c5strong a-k7 c-k7 tg-k5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --submesh-check > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"
done
rm -f gpurun_out/c5w_full.ncu-rep
echo done
