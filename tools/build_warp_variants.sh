#!/bin/bash
# Build libsilenzio variants that differ only in pbs_warp.cu's SZ_* switches:
#   tools/build_warp_variants.sh  -> tools/libsilenzio_w<DIT><TWS><ACC><POST><X32><PAD>.so for all 64 combinations
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_2504_17785_b200/build_obj
OUT=/tmp/szwv; mkdir -p $OUT
others=$(ls $OBJ/*.o | grep -v pbs_warp)
build_one() {
  local tag=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $ROOT/include --expt-relaxed-constexpr "$@" -c $ROOT/paper_2504_17785_b200/csrc/pbs_warp.cu -o $OUT/pw_$tag.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/libsilenzio_w$tag.so $others $OUT/pw_$tag.o -lcudart
}
n=0
for pad in 0 1; do for dit in 0 1; do for tws in 0 1; do for acc in 0 1; do for post in 0 1; do for x32 in 0 1; do
  tag=$dit$tws$acc$post$x32$pad
  build_one $tag -DSZ_DFT_DIT=$dit -DSZ_TW_SMEM=$tws -DSZ_ACC_FAST=$acc -DSZ_INV_TW_POST=$post -DSZ_MAC_X32=$x32 -DSZ_PAD=$pad &
  n=$((n+1)); if [ $((n % 8)) -eq 0 ]; then wait; fi
done; done; done; done; done; done
wait
ls $ROOT/tools/libsilenzio_w*.so | wc -l
