# forward projection reads geometry planes evict-first: A/B at C2 (x3) and C3
AB_ROUNDS=3 AB_VARIANTS="build/variants/cur5b.so build/variants/geomcs.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c3" AB_VARIANTS="build/variants/cur5b.so build/variants/geomcs.so" bash tools/ab.sh
