# scatter reads its tile records evict-first: A/B at C2 and C4
AB_ROUNDS=3 AB_VARIANTS="build/variants/cur3b.so build/variants/scs.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c4 --steps 5 --warmup 3" AB_VARIANTS="build/variants/cur3b.so build/variants/scs.so" bash tools/ab.sh
