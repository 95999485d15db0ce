timeout 900 python -m pytest tests/test_gpu_raster_fused.py -x -q -s 2>&1 | tail -6
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_sep.json 2>/dev/null
BS_RASTER_FUSED=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_fused.json 2>/dev/null
for f in sep fused; do python -c "import json; d=json.load(open('gpurun_out/ab_$f.json')); print('$f', d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"; done
