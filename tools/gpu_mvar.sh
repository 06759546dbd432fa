# matrix-apply variants (development aid)
export PYTHONPATH=$PWD
KS=${KS:-1,3,7,10}
echo "default (U=8, NS=3)"; python tools/matrix_based.py --ks $KS 2>&1 | python -c "import sys,json; [print(r['k'], round(r['matrix_apply_hbm_gbs']), round(r['matrix_apply_mdofs'],1), r['parity_matrix_vs_matrix_free']) for r in map(json.loads, sys.stdin)]"

for v in variants/*.so; do echo $v; DG_LIB=$PWD/$v python tools/matrix_based.py --ks $KS 2>&1 | python -c "import sys,json; [print(r['k'], round(r['matrix_apply_hbm_gbs']), round(r['matrix_apply_mdofs'],1)) for r in map(json.loads, sys.stdin)]"; done
python tools/copy_bw.py 2>&1 | tail -2
