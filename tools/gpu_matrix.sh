# NEXT-4: matrix-based tests and the comparison sweep
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matrix.py -x -q 2>&1 | tail -5
timeout 1200 python tools/matrix_based.py ${MBARGS:---big} --out gpurun_out/matrix_based.json 2>&1 | python -c "import sys,json; [print(r['k'], round(r['matrix_apply_hbm_gbs']), round(r['matrix_apply_mdofs'],1), round(r['assembly_mdofs'],2), r['parity_matrix_vs_matrix_free'], round(r.get('ratio_matrix_free_A_over_matrix',0),1)) for r in map(json.loads, sys.stdin)]"
