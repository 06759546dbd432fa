# A/B of the current build against variants/*.so on C3 (alternating, 3 rounds)
export PYTHONPATH=$PWD
for r in 1 2 3; do
echo "cur $(python tools/quick_time.py c3 20 | tail -1)"
for v in variants/*.so; do echo "$(basename $v) $(DG_LIB=$PWD/$v python tools/quick_time.py c3 20 | tail -1)"; done
done
