# on-the-fly poroelastic near field: source groups per item
cd $GRAFT_REPO_ROOT
for G in 1 2 4 8; do echo "G=$G"; DDM_PORO_GROUPS=$G DDM_NEAR_CACHE=0 python scripts/poro_mv_probe.py 2>&1 | cut -c1-40; done
