# leaf-block Jacobi: blocks across leaf boundaries (DDM_PC_SPAN=1) and block size
cd $GRAFT_REPO_ROOT
for ch in 32 48; do
  python -c "from paper_1812_05087_b200 import build as B; B.build(defines=['DDM_PC_CHUNK=$ch'], out='/tmp/ddm_pc$ch.so', force=True)" > /dev/null 2>&1
  for sp in 0 1; do
    echo "chunk $ch span $sp"
    DDM_PC_SPAN=$sp DDM_LIB=/tmp/ddm_pc$ch.so python scripts/gmres_probe.py 2>&1 | grep "solve 2"
    DDM_PC_SPAN=$sp DDM_LIB=/tmp/ddm_pc$ch.so python scripts/march_guess.py 2>&1 | grep extrap3
  done
done
