# occupancy sweep of the 2DGS raster kernels (C3): CTAs per SM forced via __launch_bounds__
for cfg in ${CFGS:-"4 3" "5 3" "5 4" "6 3"}; do
  set -- $cfg
  BS_NVCC_EXTRA="-DBS_R2_FWD_CTAS=$1 -DBS_R2_BWD_CTAS=$2" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/sweep_r2_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_r2_$1_$2.json')); print('fwd $1 bwd $2', d['value'], {k:v['ms'] for k,v in d['stages'].items() if 'raster' in k})"
done
