# sweep of the fused raster kernel: kept-list capacity, CTAs per SM, loss barrier
for cfg in ${CFGS:-"128 4 1" "128 4 0" "64 4 1" "64 5 1" "256 2 1"}; do
  set -- $cfg
  BS_NVCC_EXTRA="-DBS_FUSED_KEEP=$1 -DBS_FUSED_CTAS=$2 -DBS_FUSED_NOBAR=$3" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  BS_RASTER_FUSED=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/sweep_fused_$1_$2_$3.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_fused_$1_$2_$3.json')); print('keep $1 ctas $2 nobar $3', d['value'], d['stages']['raster']['ms'])"
done
python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
BS_RASTER_FUSED=1 timeout 600 python -m pytest tests/test_gpu_raster_fused.py -x -q 2>&1 | tail -2
