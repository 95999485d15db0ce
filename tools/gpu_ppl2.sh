BS_RASTER_PPL=2 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ppl2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ppl2.json')); print('ppl2', d['value'], {k:v['ms'] for k,v in d['stages'].items()})"
