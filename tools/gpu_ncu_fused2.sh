# ncu --set full of the fused raster kernels at C2 (3DGS) and C3 (2DGS)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"raster_fused" -c 1 -o gpurun_out/fused3_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fused3_full.log 2>&1; echo "c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"raster2d_fused" -c 1 -o gpurun_out/fused2_full \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fused2_full.log 2>&1; echo "c3 rc=$?"
