# register-resident kernels (dg_reg.cuh): GPU suite, C4 / Problem A at k = 1, 2 against the pencil kernels
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c4-k1 c4-k2 a-k1 a-k2; do
echo "reg $c $(python tools/quick_time.py $c 5 | tail -1)"
echo "pencil $c $(DG_CELL_KERNEL=pencil python tools/quick_time.py $c 5 | tail -1)"
done
