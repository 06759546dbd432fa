# Round-end refresh: GPU suite, bench line, launch list, ncu captures, sweeps, matrix-based table
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 3 -c 1 -o gpurun_out/cell_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu C3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dg_gen_kernel -s 2 -c 1 -o gpurun_out/gen_full python tools/quick_time.py a-k7 2 > gpurun_out/ncu_gen.log 2>&1; echo "ncu A-k7 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dg_reg_kernel -s 2 -c 1 -o gpurun_out/reg_a1_full python tools/quick_time.py a-k1 2 > gpurun_out/ncu_reg_a1.log 2>&1; echo "ncu A-k1 rc=$?"
python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
for k in 1 2 3 4 5 6 7 8 9 10; do echo "a-k$k $(python tools/quick_time.py a-k$k 5 | tail -1)"; done | tee gpurun_out/problemA.log
python tools/matrix_based.py --big --out gpurun_out/matrix_based.json > gpurun_out/matrix.log 2>&1; echo "matrix rc=$?"
for k in 1 2 3 4 5 6 7 8; do echo "tg-k$k $(python tools/quick_time.py tg-k$k 3 | tail -1)"; done | tee gpurun_out/tg.log
