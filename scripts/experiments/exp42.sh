# GMRES: finish + normalise + next leaf-block apply fused
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_precond.py tests/test_gpu_knobs.py -x -q 2>&1 | tail -1
python scripts/gmres_probe.py 2>&1 | grep "solve 2"
DDM_GMRES_FUSE_PC=0 python scripts/gmres_probe.py 2>&1 | grep "solve 2"
python scripts/march_guess.py 2>&1 | grep extrap3
DDM_GMRES_FUSE_PC=0 python scripts/march_guess.py 2>&1 | grep extrap3
