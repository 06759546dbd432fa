export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "c3 $(python tools/quick_time.py c3 10 | tail -1)"
echo "a-k7 tma   $(python tools/quick_time.py a-k7 5 | tail -1)"
echo "a-k7 notma $(DG_NO_TMA=1 python tools/quick_time.py a-k7 5 | tail -1)"
