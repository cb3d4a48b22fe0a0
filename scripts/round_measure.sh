# GPU test suite + bench line + launch list + ncu --set full captures of one
# config-5 matvec's kernels (serial schedule) and of bbFMM n = 6.
# Usage (GPU box): bash scripts/round_measure.sh [tag]   (outputs in gpurun_out/)
cd $GRAFT_REPO_ROOT
tag=${1:-r2}
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
DDM_SERIAL=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"prep_stream|p2p_leaf_kernel|p2m_kernel|m2m_|m2l_kernel|l2l_|l2p_block|finalize_near" -c 40 -o gpurun_out/${tag}_step python scripts/profile_matvec.py 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bb_" -c 12 -o gpurun_out/${tag}_bb6 python scripts/profile_matvec.py 1 20 5 bbfmm6 > gpurun_out/ncu_bb.log 2>&1; echo "ncu bb rc=$?"
