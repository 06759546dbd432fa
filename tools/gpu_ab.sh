# A/B of the current build against variants/*.so (alternating, 3 rounds) on the workloads in $WL (default c3)
export PYTHONPATH=$PWD
for r in 1 2 3; do
for w in ${WL:-c3}; do
echo "cur $w $(python tools/quick_time.py $w ${REPS:-20} | tail -1)"
for v in variants/*.so; do echo "$(basename $v) $w $(DG_LIB=$PWD/$v python tools/quick_time.py $w ${REPS:-20} | tail -1)"; done
done
done
