# one --set full capture of the fused projection backward + Adam (C2) with source counters
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"project_bwd_adam" -c 1 -o gpurun_out/adam_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/adam_full.log 2>&1
