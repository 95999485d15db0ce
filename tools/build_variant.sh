#!/bin/bash
# build/variants/<name>.so: libsplat_b200.so with raster sources compiled with extra flags (A/B tuning)
# usage: tools/build_variant.sh NAME "-DFLAG=1 ..." [src.cu ...]
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; shift 2; srcs=${@:-raster.cu}
mkdir -p build/variants/$name.obj
objs=""
for o in paper_2512_20017_b200/_lib/obj/*.o; do
  b=$(basename $o .o)
  if [[ " $srcs " == *" $b.cu "* ]]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr $flags -c paper_2512_20017_b200/csrc/$b.cu -o build/variants/$name.obj/$b.o
    objs="$objs build/variants/$name.obj/$b.o"
  else
    objs="$objs $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so $objs -lcudart
echo build/variants/$name.so
