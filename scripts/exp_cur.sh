python scripts/tune.py base DDM_LEAF_TPL=3 "DDM_LEAF_TPL=3,DDM_LEAF_MINB=5" "DDM_LEAF_TPL=3,DDM_LEAF_UNROLL=1" "DDM_LEAF_TPL=4,DDM_LEAF_MINB=4" 2>&1 | grep -v Warn
TUNE_SERIAL=0 python scripts/tune.py base DDM_LEAF_TPL=3 2>&1 | grep -v Warn
