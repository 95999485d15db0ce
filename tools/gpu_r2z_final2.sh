# round-2 closing evidence: GPU suite, smoke, bench C2 (with CPU baseline) / C3 / C4, reference arm, sanitizers
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2z2_pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2z2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2z2_smoke.log
timeout 900 python bench.py > gpurun_out/r2z2_bench_c2.json 2> gpurun_out/r2z2_bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r2z2_bench_c3.json 2> gpurun_out/r2z2_bench_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2z2_bench_c4.json 2> gpurun_out/r2z2_bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2z2_bench_reference.json 2> gpurun_out/r2z2_bench_reference.err; echo "ref rc=$?"
for f in c2 c3 c4; do python -c "import json; d=json.load(open('gpurun_out/r2z2_bench_$f.json')); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['binding'], (d['roofline'].get('issue') or {}).get('frac'), d['roofline']['step_hbm']['frac'], (d.get('cpu_baseline') or {}).get('value'), {k:v['ms'] for k,v in d['stages'].items()})"; done
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2z2_bench_c2_2ranks_one_gpu.json 2> gpurun_out/r2z2_bench_c2_2ranks.err; echo "2 ranks rc=$?"; head -c 600 gpurun_out/r2z2_bench_c2_2ranks_one_gpu.json

timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scatter_rec|sort_tiles" -c 3 -o gpurun_out/r2z2_full_c2 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2z2_full_c2.log 2>&1; echo "full c2 rc=$?"
