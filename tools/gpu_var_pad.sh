# constant-bank placement sweep: variants/n<N>_padx<X>.so against the default, C4 and Problem A at k = N-1
export PYTHONPATH=$PWD
for n in 4 5 6 7 9 10 11; do k=$((n-1));
echo "default n$n c4 $(python tools/quick_time.py c4-k$k 5 | tail -1) a $(python tools/quick_time.py a-k$k 3 | tail -1)"
for v in variants/n${n}_*.so; do echo "$(basename $v) c4 $(DG_LIB=$PWD/$v python tools/quick_time.py c4-k$k 5 | tail -1) a $(DG_LIB=$PWD/$v python tools/quick_time.py a-k$k 3 | tail -1)"; done
done
