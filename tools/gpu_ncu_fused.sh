timeout 600 ncu --set full --clock-control none --import-source on -k regex:"raster_fused" -c 1 -o gpurun_out/fused_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fused_full.log 2>&1
