# C4 timings of the default build and of every variant in variants/ (n<N>_... -> c4-k<N-1>)
export PYTHONPATH=$PWD
for k in ${KS:-1 2 3 4 5 6 8 9 10}; do echo "default c4-k$k $(python tools/quick_time.py c4-k$k 5 | tail -1)"; done
for v in variants/*.so; do n=$(basename $v | sed -E 's/^n([0-9]+)_.*/\1/'); k=$((n-1)); echo "$(basename $v) c4-k$k $(DG_LIB=$PWD/$v python tools/quick_time.py c4-k$k 5 | tail -1)"; done
