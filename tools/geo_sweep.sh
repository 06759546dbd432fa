# Multilinear-geometry (Problem C stand-in) and over-integration timing sweep (run under gpurun)
export PYTHONPATH=$PWD
for k in 1 2 3 4 5 6 7 8 9 10; do echo "c-k$k $(python tools/quick_time.py c-k$k 5 | tail -1)"; done
