export DG_CELL_KERNEL=mma
python tools/quick_time.py c3 10 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:dg_cell_mma8 -s 2 -c 1 -o gpurun_out/mma_full python tools/quick_time.py c3 3 > gpurun_out/ncu_mma.log 2>&1; echo "ncu rc=$?"
