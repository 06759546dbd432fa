export PYTHONPATH=$PWD
python tools/quick_time.py a-k7 5 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:dg_gen_kernel -s 2 -c 1 -o gpurun_out/gen_full python tools/quick_time.py a-k7 2 > gpurun_out/ncu_gen.log 2>&1; echo "ncu rc=$?"
