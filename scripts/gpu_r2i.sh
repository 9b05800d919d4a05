# dtw4: finvar only for L > 256, reorder off; reverse cumulative bound at narrow bands (TSW_CENV_DP)
bash scripts/ab.sh "2:dtw 3:dtw 5:dtw" 2 "base=TSW_LIB=build_var/base/libtswarp_b200.so" "cur=X=1" "cenvdp=TSW_CENV_DP=1"
