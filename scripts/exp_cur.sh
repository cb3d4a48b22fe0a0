nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rcp_probe scripts/micro/rcp_probe.cu && /tmp/rcp_probe
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2P_RCP2=1 base DDM_P2P_RCP2=1 2>&1 | grep -v Warn
