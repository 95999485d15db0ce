# round-2 final evidence at HEAD: GPU suite, smoke, bench C2 (with CPU baseline) / C3 / C4, reference arm,
# C2 + C4 launch lists, ncu --set full of the hot kernels of C2 and C3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2y_pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2y_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2y_smoke.log
timeout 900 python bench.py > gpurun_out/r2y_bench_c2.json 2> gpurun_out/r2y_bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2y_bench_c3.json 2> gpurun_out/r2y_bench_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2y_bench_c4.json 2> gpurun_out/r2y_bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2y_bench_reference.json 2> gpurun_out/r2y_bench_reference.err; echo "ref rc=$?"
for f in c2 c3 c4; do python -c "import json; d=json.load(open('gpurun_out/r2y_bench_$f.json')); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['binding'], d['roofline']['step_hbm']['frac'], (d.get('cpu_baseline') or {}).get('value'), {k:v['ms'] for k,v in d['stages'].items()})"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r2y_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_launches_c2.log 2>&1; echo "launches c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y_launches_c4.csv \
    python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_launches_c4.log 2>&1; echo "launches c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"cull_kernel|project_fwd|scatter_rec|sort_tiles|raster_fused|project_bwd_adam" \
    -c 8 -o gpurun_out/r2y_full_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_full_c2.log 2>&1; echo "full c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"raster2d_fused|project_bwd_adam" -c 2 -o gpurun_out/r2y_full_c3 \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_full_c3.log 2>&1; echo "full c3 rc=$?"
ls -la gpurun_out/ | grep r2f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cull_kernel" -c 1 -o gpurun_out/r2y_full_c4_cull \
    python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_full_c4_cull.log 2>&1; echo "full c4 cull rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_fwd|project_bwd_adam|list_chunks" -c 3 -o gpurun_out/r2y_full_c4_proj \
    python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_full_c4_proj.log 2>&1; echo "full c4 proj rc=$?"
python tools/timeline.py --steps 3 --e2e > gpurun_out/r2y_timeline_e2e_c2.txt 2>&1; echo "timeline rc=$?"
SAN_PREFIX=r2y bash tools/sanitize.sh
