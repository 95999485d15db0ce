# round-2 evidence at HEAD: ncu launch list + --set full (C2, C3), sanitizers, GPU suite, smoke, bench lines, reference arm
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r2_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_launches_c2.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"cull_kernel|project_fwd|scatter_rec|sort_tiles|raster_fused|project_bwd_adam" \
    -c 8 -o gpurun_out/r2_full_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_full_c2.log 2>&1
BS_RASTER_FUSED=0 ncu --set full --clock-control none -k regex:"raster_fwd|raster_bwd" \
    -c 2 -o gpurun_out/r2_full_c2_separate python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_full_c2s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"raster2d|project_bwd_adam" -c 2 -o gpurun_out/r2_full_c3 \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_full_c3.log 2>&1
bash tools/sanitize.sh
