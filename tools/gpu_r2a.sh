# round-2 check: new parity tests (verbose), whole GPU suite, C2 bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_fused_adam.py tests/test_gpu_fullscale.py tests/test_kat.py -m gpu -q -rA -s \
    > gpurun_out/r2a_newtests.log 2>&1; echo "newtests rc=$?"
tail -30 gpurun_out/r2a_newtests.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2a_gpu_all.log 2>&1; echo "all rc=$?"
tail -15 gpurun_out/r2a_gpu_all.log
timeout 600 python bench.py > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err; echo "bench rc=$?"
tail -3 gpurun_out/r2a_bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/r2a_bench_c2.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['step_hbm'], {k:(v['ms'],v['hbm_frac'],v['issue_frac']) for k,v in d['stages'].items()})"
