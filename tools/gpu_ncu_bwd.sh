# one --set full capture of the product raster_bwd (C2) with source counters
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"raster_bwd|raster_fwd" -c 2 -o gpurun_out/bwd_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bwd_full.log 2>&1
