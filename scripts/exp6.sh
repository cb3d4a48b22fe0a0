cd $GRAFT_REPO_ROOT
for v in DDM_SRC_CHUNK=128 DDM_SRC_CHUNK=32 DDM_SRC_CHUNK=16; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_05087_b200 import build as B
B.build(defines=['$v'], out='/tmp/var.so', force=True)"
  echo $v; DDM_LIB=/tmp/var.so python scripts/poro_timing.py | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(k, round(v['matvec_ms'],3), round(v['stages_serial_ms']['p2p'],3), v['tree']['P2P_ITEMS'])"
done 2>&1 | tee -a gpurun_out/exp6.log
DDM_SERIAL=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:poro_p2p -c 1 -o gpurun_out/porop2p python scripts/poro_timing.py > /dev/null 2>&1
