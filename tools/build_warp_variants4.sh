#!/bin/bash
# Round-1 fourth sweep (SZ_PAD = 0): SZ_TAN_TWIST{1,2,3} x SZ_ACC_CQ{4,8} x SZ_MAC_X32 x SZ_INV_TW_POST
#   -> tools/libsilenzio_y<TAN><CQ><X32><POST>.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_2504_17785_b200/build_obj
OUT=/tmp/szwv4; mkdir -p $OUT
others=$(ls $OBJ/*.o | grep -v pbs_warp)
build_one() {
  local tag=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $ROOT/include --expt-relaxed-constexpr "$@" -c $ROOT/paper_2504_17785_b200/csrc/pbs_warp.cu -o $OUT/pw_$tag.o 2>/dev/null
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/libsilenzio_y$tag.so $others $OUT/pw_$tag.o -lcudart
}
n=0
for tan in 1 2 3; do for cq in 4 8; do for x32 in 0 1; do for post in 0 1; do
  build_one $tan$cq$x32$post -DSZ_PAD=0 -DSZ_TAN_TWIST=$tan -DSZ_ACC_CQ=$cq -DSZ_MAC_X32=$x32 -DSZ_INV_TW_POST=$post &
  n=$((n+1)); if [ $((n % 8)) -eq 0 ]; then wait; fi
done; done; done; done
wait
ls $ROOT/tools/libsilenzio_y*.so | wc -l
