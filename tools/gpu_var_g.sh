export PYTHONPATH=$PWD
for k in 4 5 7 8 9; do echo "default a-k$k $(python tools/quick_time.py a-k$k 5 | tail -1)"; done
for v in variants/*.so; do n=$(basename $v | sed -E 's/^g([0-9]+)_.*/\1/'); k=$((n-1)); echo "$(basename $v) a-k$k $(DG_LIB=$PWD/$v python tools/quick_time.py a-k$k 5 | tail -1)"; done
