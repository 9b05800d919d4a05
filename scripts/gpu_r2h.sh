# which dtw4 diet change costs C2/C3: same-box A/B of the variants
bash scripts/ab.sh "2:dtw 3:dtw 5:dtw" 2 "base=TSW_LIB=build_var/base/libtswarp_b200.so" "cur=X=1" "noidle=TSW_DTW4_NOIDLE=1" "noreorder=TSW_LIB=build_var/noreorder/libtswarp_b200.so" "nofinvar=TSW_LIB=build_var/nofinvar/libtswarp_b200.so"
