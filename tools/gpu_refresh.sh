# Refresh of the committed evidence on one B200 (run under gpurun): GPU suite, bench lines,
# launch list, ncu --set full captures of the operator kernels, degree / workload sweeps.
# Every ncu command follows a plain run of the same command that exited 0 (B200_PROFILING.md).
# The captures are summarised on the box (tools/ncu_summary.py) before the bench lines run; copy
# gpurun_out/ncu_full_summary.json to profiles/ afterwards.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
# captures first (fresh clocks), each after its plain run
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
# summaries of the captures (this build's kernel hashes), so the bench lines below carry the roofline
for a in "c3_full C3 268435456" "c5w_full C5-weak-P1 536870912" "c4-k8_full C4-k8 102503232" "c4-k10_full C4-k10 98611128" "a-k7_full A-k7 398688256" "c-k7_full C-k7 398688256" "tg-k5_full TG-k5 401947272"; do
  set -- $a; [ -f gpurun_out/$1.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$1.ncu-rep --name $2 --ndofs $3 --json profiles/ncu_full_summary.json > /dev/null
done
cp profiles/ncu_full_summary.json gpurun_out/ncu_full_summary.json
# bench lines
python bench.py --steps 20 --warmup 5 --submesh-check > gpurun_out/bench_c3.log 2>&1; echo "bench C3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-200
for w in c5weak c5strong a-k7 c-k7 tg-k5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --submesh-check > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "reference rc=$?"
# the N-rank path (torch.distributed.run, IPC face-trace halo) with 8 ranks sharing this GPU: not a scaling number
python bench.py --gpus 8 --share-gpu --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_share8.log 2>&1; echo "share8 rc=$?"
# sweeps
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
for k in 1 2 3 4 5 6 7 8 9 10; do echo "a-k$k $(python tools/quick_time.py a-k$k 5 | tail -1)"; done > gpurun_out/problemA.log
for k in 1 2 3 4 5 6 7 8 9 10; do echo "tg-k$k $(python tools/quick_time.py tg-k$k 3 | tail -1)"; done > gpurun_out/tg.log
bash tools/geo_sweep.sh > gpurun_out/geo.log 2>&1
echo done
