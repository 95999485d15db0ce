timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_hbm']['frac'])"
