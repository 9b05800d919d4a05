# Build a variant of the library with extra -D flags on the DTW/DK kernel files:
#   bash scripts/build_variant.sh NAME "-DFOO=0 -DBAR=1" [files...]   -> build_var/NAME/libtswarp_b200.so
set -e
NAME=$1; DEFS=$2; shift 2; FILES=${@:-kernels_dtw4.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd); CS=$ROOT/paper_1811_11076_b200/csrc; OBJ=$ROOT/paper_1811_11076_b200/lib/obj
OUT=$ROOT/build_var/$NAME; mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-O3,-ffp-contract=off -I$ROOT/include"
objs=""
for o in $OBJ/*.o; do
  b=$(basename $o .o); skip=0
  for f in $FILES; do [ "$b" = "${f%.cu}" ] && skip=1; done
  [ $skip = 0 ] && objs="$objs $o"
done
for f in $FILES; do $NV $DEFS -c -o $OUT/${f%.cu}.o $CS/$f; objs="$objs $OUT/${f%.cu}.o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $OUT/libtswarp_b200.so $objs -lpthread
echo built $OUT/libtswarp_b200.so
