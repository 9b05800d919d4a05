bash scripts/ab.sh "2:dtw 3:dtw 5:dtw" 2 "base=TSW_LIB=build_var/base/libtswarp_b200.so" "cur=X=1" "nolb2=TSW_LB2=0,TSW_CENV_DP=1"
