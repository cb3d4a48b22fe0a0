# targets per P2P work item (16 vs 32) and sources per item
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_TGT_GROUP=32 DDM_TGT_GROUP=32,DDM_SRC_CHUNK=1024 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base DDM_TGT_GROUP=32 2>&1 | grep total
