# register-resident kernel (dg_reg.cuh, n <= 3): GPU suite, C4 k = 1, 2 against the pencil kernel, ncu capture
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 1 2; do
echo "reg k$k $(python tools/quick_time.py c4-k$k 5 | tail -1)"
echo "pencil k$k $(DG_CELL_KERNEL=pencil python tools/quick_time.py c4-k$k 5 | tail -1)"
ncu --set full --clock-control none --import-source on -k regex:dg_reg_kernel -s 2 -c 1 -o gpurun_out/reg_k${k}_full python tools/quick_time.py c4-k$k 2 > gpurun_out/ncu_reg_k$k.log 2>&1; echo "ncu k$k rc=$?"
done
