# Problem A timings of the default build and of the variants in variants/g<N>_... (-> a-k<N-1>)
export PYTHONPATH=$PWD
for k in ${KS:-2}; do echo "default a-k$k $(DG_CELL_KERNEL=${DGK:-} python tools/quick_time.py a-k$k 5 | tail -1)"; done
for v in variants/*.so; do n=$(basename $v | sed -E 's/^g([0-9]+)_.*/\1/'); k=$((n-1)); echo "$(basename $v) a-k$k $(DG_LIB=$PWD/$v python tools/quick_time.py a-k$k 5 | tail -1)"; done
