cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_SRC_CHUNK=128 DDM_SRC_CHUNK=64 DDM_SRC_CHUNK=32 2>&1 | tee gpurun_out/exp5.log
for v in DDM_SRC_CHUNK=128 DDM_SRC_CHUNK=64 DDM_SRC_CHUNK=32; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_05087_b200 import build as B
B.build(defines=['$v'], out='/tmp/var.so', force=True)"
  echo $v; DDM_LIB=/tmp/var.so python scripts/poro_timing.py | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(k, round(v['matvec_ms'],3), round(v['stages_serial_ms']['p2p'],3), v['tree']['P2P_ITEMS'])"
done 2>&1 | tee -a gpurun_out/exp5.log
