TSW_DEBUG_WATCH=1 timeout 120 python scripts/diag_big_values.py > gpurun_out/r2g_diag.log 2>&1; echo "diag rc=$?"; tail -30 gpurun_out/r2g_diag.log
