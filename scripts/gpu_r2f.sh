# dtw4: +inf idle lanes, reordered mins, last-body fin capture, reverse cumulative bound.
# GPU tests with a per-test timeout (find the slow / hanging one), then same-box A/B.
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 420 --durations 12 > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"; tail -20 gpurun_out/r2f_pytest.log
bash scripts/ab.sh "2:dtw 3:dtw 5:dtw" 2 "base=TSW_LIB=build_var/base/libtswarp_b200.so" "norev=TSW_REVCB=0" "cur=X=1"
