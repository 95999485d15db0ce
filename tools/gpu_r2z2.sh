# evict-first Adam hints: fused-Adam parity tests, A/B at C2 and C3 (0 = none, 1 = moments ld/st + param st, 2 = stores only), C4 with the default
timeout 900 python -m pytest tests/test_gpu_fused_adam.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2z_pytest_adam.log 2>&1; echo "adam tests rc=$?"; tail -2 gpurun_out/r2z_pytest_adam.log
AB_ROUNDS=3 AB_VARIANTS="build/variants/base0.so build/variants/stream1.so build/variants/stream2.so" bash tools/ab.sh
AB_ROUNDS=2 AB_ARGS="--config c3" AB_VARIANTS="build/variants/base0.so build/variants/stream1.so" bash tools/ab.sh
timeout 1500 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2z_bench_c4.json 2> gpurun_out/r2z_bench_c4.err; echo "c4 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2z_bench_c4.json')); print('c4', d['value'], d['e2e']['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
