# tuning probe: raster_bwd time without the gradient reduction (upper bound of any reduction scheme)
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/probe_base.json 2>/dev/null
BS_NVCC_EXTRA="-DBS_BWD_NO_REDUCE" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/probe_noreduce.json 2>/dev/null
for f in base noreduce; do python -c "import json; d=json.load(open('gpurun_out/probe_$f.json')); print('$f', d['value'], {k:v['ms'] for k,v in d['stages'].items() if 'raster' in k})"; done
