BS_NVCC_EXTRA=-DBS_RASTER_STATS python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
timeout 600 python tools/raster_stats.py 3dgs
BS_RASTER_FUSED=0 timeout 600 python tools/raster_stats.py 3dgs
python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
