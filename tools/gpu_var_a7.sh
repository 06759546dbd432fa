export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_next1.py -x -q 2>&1 | tail -1
echo "default $(python tools/quick_time.py a-k7 5 | tail -1)"
for v in variants/*.so; do echo "$(basename $v) $(DG_LIB=$PWD/$v python tools/quick_time.py a-k7 5 | tail -1)"; done
