# round-2 check: GPU suite + C2 / C3 bench lines (no CPU baseline)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2b_gpu_all.log 2>&1; echo "all rc=$?"
tail -4 gpurun_out/r2b_gpu_all.log
for c in c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2b_bench_$c.json 2> gpurun_out/r2b_bench_$c.err; echo "bench $c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r2b_bench_$c.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['step_hbm']['frac'], {k:(v['ms'],v['hbm_frac'],v['issue_frac']) for k,v in d['stages'].items()})"
done
