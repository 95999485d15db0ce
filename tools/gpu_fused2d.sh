timeout 900 python -m pytest tests/test_gpu_raster_fused.py -x -q -s 2>&1 | tail -4
BS_RASTER_FUSED=0 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/c3_sep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/c3_sep.json')); print('sep', d['value'], {k:v['ms'] for k,v in d['stages'].items()})"
for cfg in ${CFGS:-"64 3" "128 3" "32 4"}; do
  set -- $cfg
  BS_NVCC_EXTRA="-DBS_FUSED2_KEEP=$1 -DBS_FUSED2_CTAS=$2" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/c3_fused_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c3_fused_$1_$2.json')); print('keep $1 ctas $2', d['value'], {k:v['ms'] for k,v in d['stages'].items()})"
done
python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
