# node-sharing stream: new geometry tests + ncu full of the stream p2p kernel and prep
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py -x -q -k "node_sharing or small_and_single or cfg5" 2>&1 | tail -3 | tee gpurun_out/exp17.log
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"p2p_kernel|prep_stream" -c 2 -o gpurun_out/full_p2p_stream python scripts/profile_matvec.py 1 > gpurun_out/ncu_p2p.log 2>&1; echo "ncu rc=$?" | tee -a gpurun_out/exp17.log
