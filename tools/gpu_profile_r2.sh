# ncu evidence (round 2): launch list of C2 steps, --set full of the hot kernels of one C2 step and of C3
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r2_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_launches_c2.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"cull_kernel|project_fwd|count_tiles|scatter_tiles|scatter_rec|sort_tiles|raster_fwd|raster_bwd|project_bwd_adam" \
    -c 12 -o gpurun_out/r2_full_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_full_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"raster2d|project_bwd_adam" -c 3 -o gpurun_out/r2_full_c3 \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_full_c3.log 2>&1
ls -la gpurun_out/
