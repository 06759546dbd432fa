#!/bin/bash
# Time every variants/n<N>_*.so on C4 at k = N-1 (and the default build) -- development aid.
export PYTHONPATH=$PWD
for n in $(ls variants | sed -E 's/^n([0-9]+)_.*/\1/' | sort -un); do
  k=$((n-1))
  echo "n=$n default $(python tools/quick_time.py c4-k$k 5 | tail -1)"
  for v in variants/n${n}_*.so; do
    echo "n=$n $(basename $v .so) $(DG_LIB=$PWD/$v python tools/quick_time.py c4-k$k 5 | tail -1)"
  done
done
