#!/bin/bash
# A/B the prebuilt variants build/variants/*.so on one box: alternate them R times,
# C2 (and C3 if AB_C3=1) bench lines, raster stage ms; restores the in-tree library at the end
cd "$(dirname "$0")/.."
lib=paper_2512_20017_b200/_lib/libsplat_b200.so
cp $lib /tmp/libsplat_b200.orig.so
for r in $(seq 1 ${AB_ROUNDS:-3}); do
  for v in ${AB_VARIANTS:-$(ls build/variants/*.so)}; do
    cp $v $lib
    n=$(basename $v .so)
    timeout 300 python bench.py --no-cpu-baseline --steps 20 ${AB_ARGS} > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
    python -c "import json; d=json.load(open('gpurun_out/ab_$n.json')); print('$n', d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
  done
done
cp /tmp/libsplat_b200.orig.so $lib
