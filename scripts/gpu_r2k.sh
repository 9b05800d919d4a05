timeout 600 python -m pytest tests/test_cli_metrics.py -q -m gpu -x --timeout 300 > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k_pytest.log
bash scripts/ab.sh "2:dtw 3:dtw 5:dtw" 2 "cur=X=1" "rtlong=TSW_LIB=build_var/rtlong/libtswarp_b200.so"
