# projection L2 hints: SH staged evict-first (both projection kernels), G_SP clear with st.cs; A/B at C2 and C3
AB_ROUNDS=3 AB_VARIANTS="build/variants/cur2b.so build/variants/shef.so build/variants/zcs.so build/variants/shef_zcs.so" bash tools/ab.sh
AB_ROUNDS=1 AB_ARGS="--config c3" AB_VARIANTS="build/variants/cur2b.so build/variants/shef.so build/variants/zcs.so build/variants/shef_zcs.so" bash tools/ab.sh
