# bucket sorts read their keys evict-first: A/B at C2 (x4) and C3
AB_ROUNDS=4 AB_VARIANTS="build/variants/cur4b.so build/variants/sortcs.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c3" AB_VARIANTS="build/variants/cur4b.so build/variants/sortcs.so" bash tools/ab.sh
