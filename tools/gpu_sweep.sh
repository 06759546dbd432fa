# C4 degree sweep + C2/C3/C5 through tools/sweep.py, and the C3 bench line
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python tools/sweep.py --out gpurun_out/sweep.json 2>&1 | tail -16
