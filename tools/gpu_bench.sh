# bench lines only: bash tools/gpu_bench.sh <tag> <config>...
tag=$1; shift
for c in "$@"; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err; echo "bench $c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/${tag}_bench_$c.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['step_hbm']['frac'], {k:(v['ms'],v['hbm_frac'],v['issue_frac']) for k,v in d['stages'].items()})"
done
