# full ncu captures of the fast kernel at k = 4, 8, 10 (C4)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for k in 4 8 10; do
ncu --set full --clock-control none --import-source on -k regex:dg_cell_kernel -s 2 -c 1 -o gpurun_out/c4k${k}_full python tools/quick_time.py c4-k$k 2 > gpurun_out/ncu_k$k.log 2>&1; echo "ncu k$k rc=$?"
done
