export PYTHONPATH=$PWD
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 1 2 3 4 5 6 7 8 9 10; do echo "a-k$k $(python tools/quick_time.py a-k$k 5 | tail -1)"; done
