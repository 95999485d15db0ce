# fused raster changes: tests, racecheck of the small step, bench C2/C3/C4
timeout 900 python -m pytest tests/test_gpu_raster_fused.py tests/test_gpu_parity.py tests/test_kat.py tests/test_gpu_work_list.py tests/test_gpu_fullscale.py -q -x 2>&1 | tail -1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --target-processes all python tools/sanitize_step.py > gpurun_out/rc_check.log 2>&1; tail -1 gpurun_out/rc_check.log
unset PYTORCH_NO_CUDA_MEMORY_CACHING
for c in c2 c3 c4; do python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['primitive'], d['value'], d['e2e']['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"; done
