# sparse-RED lane threshold of the backward, swept in the fused raster kernel (C2)
for L in ${LANES:-8 12 14 16 20}; do
  BS_NVCC_EXTRA="-DBS_SPARSE_LANES=$L" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/sweep_sparse_fused_$L.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_sparse_fused_$L.json')); print('lanes $L', d['value'], d['stages']['raster']['ms'])"
done
python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/sweep_sparse_fused_10.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/sweep_sparse_fused_10.json')); print('lanes 10', d['value'], d['stages']['raster']['ms'])"
