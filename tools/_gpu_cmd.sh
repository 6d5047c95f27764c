cd $GRAFT_REPO_ROOT
O=gpurun_out
CONFIGS="5 3 2" bash tools/ab.sh libcbvh_cur.so libcbvh_nozs.so libcbvh_pre_zs.so libcbvh_cur.so > $O/r2_ab_zsbranch.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "error_paths or zero_suppressed or staging" > $O/r2_gputest5.log 2>&1; echo "pytest rc=$?" >> $O/r2_gputest5.log
