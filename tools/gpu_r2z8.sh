# fused Adam prefetches one round ahead: A/B at C2 (x3), C3, C4
AB_ROUNDS=3 AB_VARIANTS="build/variants/cur6b.so build/variants/pfnext.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c3" AB_VARIANTS="build/variants/cur6b.so build/variants/pfnext.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c4 --steps 5 --warmup 3" AB_VARIANTS="build/variants/cur6b.so build/variants/pfnext.so" bash tools/ab.sh
