#!/bin/bash
# Round-1 third sweep (SZ_ACC_CQ = 4): SZ_PAD x SZ_TW_SMEM x SZ_D_ST32 x SZ_TAN_TWIST{0,2}
#   -> tools/libsilenzio_x<PAD><TWS><DST><TAN>.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_2504_17785_b200/build_obj
OUT=/tmp/szwv3; mkdir -p $OUT
others=$(ls $OBJ/*.o | grep -v pbs_warp)
build_one() {
  local tag=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $ROOT/include --expt-relaxed-constexpr "$@" -c $ROOT/paper_2504_17785_b200/csrc/pbs_warp.cu -o $OUT/pw_$tag.o 2>/dev/null
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/libsilenzio_x$tag.so $others $OUT/pw_$tag.o -lcudart
}
n=0
for pad in 0 1; do for tws in 0 1; do for dst in 0 1; do for tan in 0 2; do
  build_one $pad$tws$dst$tan -DSZ_ACC_CQ=4 -DSZ_PAD=$pad -DSZ_TW_SMEM=$tws -DSZ_D_ST32=$dst -DSZ_TAN_TWIST=$tan &
  n=$((n+1)); if [ $((n % 8)) -eq 0 ]; then wait; fi
done; done; done; done
wait
ls $ROOT/tools/libsilenzio_x*.so | wc -l
