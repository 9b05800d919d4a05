timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -k "reverse or fast_path or knn or beyond or long or lb_box_exact or concurrent" > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2l_pytest.log
bash scripts/ab.sh "5:dtw" 2 "v2=TSW_LIB=build_var/v2/libtswarp_b200.so" "cur=X=1"
