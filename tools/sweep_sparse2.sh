for L in ${LANES:-5 8 12}; do
  BS_NVCC_EXTRA="-DBS_SPARSE2_LANES=$L" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/sweep2_$L.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep2_$L.json')); print('lanes $L', d['value'], {k:v['ms'] for k,v in d['stages'].items() if 'raster' in k})"
done
