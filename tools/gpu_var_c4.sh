export PYTHONPATH=$PWD
for v in variants/*.so; do n=$(basename $v | sed -E 's/^n([0-9]+)_.*/\1/'); k=$((n-1)); echo "$(basename $v) c4-k$k $(DG_LIB=$PWD/$v python tools/quick_time.py c4-k$k 5 | tail -1)"; done
