export PYTHONPATH=$PWD
echo "default $(python tools/quick_time.py c3 10 | tail -1)"
for v in variants/*.so; do echo "$(basename $v) $(DG_LIB=$PWD/$v python tools/quick_time.py c3 10 | tail -1)"; done
