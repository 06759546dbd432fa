export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 1 2 3 4 5 6 7 8 9 10; do echo "c4-k$k $(python tools/quick_time.py c4-k$k 5 | tail -1)"; done
echo "c3 $(python tools/quick_time.py c3 10 | tail -1)"
