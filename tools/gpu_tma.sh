export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "tma   $(python tools/quick_time.py c3 10 | tail -1)"
echo "notma $(DG_NO_TMA=1 python tools/quick_time.py c3 10 | tail -1)"
echo "tma c4-k7  $(python tools/quick_time.py c4-k7 10 | tail -1)"
