#!/bin/bash
# Build a diagnostic/experimental libsilenzio variant with extra -D flags:
#   tools/build_variant.sh NAME -DFOO -DBAR   -> tools/libsilenzio_NAME.so
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=/tmp/szvar_$NAME; mkdir -p $OUT
for f in $ROOT/paper_2504_17785_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $ROOT/include --expt-relaxed-constexpr "$@" -c $f -o $OUT/$(basename $f).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/libsilenzio_$NAME.so $OUT/*.o -lcudart
echo built tools/libsilenzio_$NAME.so
