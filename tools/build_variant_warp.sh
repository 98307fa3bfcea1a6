#!/bin/bash
# Fast variant build for set-A kernel experiments: recompile only pbs_warp.cu
# with extra -D flags and link it against the default build's other objects:
#   tools/build_variant_warp.sh NAME -DFOO=1   -> tools/libsilenzio_NAME.so
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_2504_17785_b200/build_obj
OUT=/tmp/szvarw_$NAME; mkdir -p $OUT
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I $ROOT/include --expt-relaxed-constexpr -Xptxas -v "$@" -c $ROOT/paper_2504_17785_b200/csrc/pbs_warp.cu \
  -o $OUT/pbs_warp.cu.o 2> $OUT/ptxas.log
grep -A1 "blind_rotate_warp_kernelILi3ELb0" $OUT/ptxas.log | grep -E "registers|spill" | head -2
others=$(ls $OBJ/*.o | grep -v pbs_warp.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/libsilenzio_$NAME.so $OUT/pbs_warp.cu.o $others -lcudart
echo built tools/libsilenzio_$NAME.so
