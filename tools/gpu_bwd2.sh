# fused raster kernels compacted kept lists + two-record backward: parity vs the two-kernel path + bench C2/C3
python -c "from paper_2512_20017_b200.build import build_native; build_native()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_raster_fused.py tests/test_gpu_fullscale.py -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2', d['value'], d['e2e']['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3', d['value'], d['e2e']['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
done
