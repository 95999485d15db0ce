# G_SP evict-first loads in the projection backward: A/B at C2/C3 vs the adopted store hints, and the DRAM bytes of each under ncu
AB_ROUNDS=3 AB_VARIANTS="build/variants/cur.so build/variants/gspcs.so build/variants/gspcs_s1.so" bash tools/ab.sh
AB_ROUNDS=2 AB_ARGS="--config c3" AB_VARIANTS="build/variants/cur.so build/variants/gspcs.so" bash tools/ab.sh
lib=paper_2512_20017_b200/_lib/libsplat_b200.so; cp $lib /tmp/orig.so
for v in base0 cur gspcs; do
  cp build/variants/$v.so $lib
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:project_bwd_adam -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2z_ncu_adam_$v.csv 2> gpurun_out/r2z_ncu_adam_$v.err; echo "ncu $v rc=$?"
  grep -E "dram__bytes|gpu__time" gpurun_out/r2z_ncu_adam_$v.csv | tail -3 | awk -F'","' '{print "'$v'", $(NF-2), $(NF-1), $NF}'
done
cp /tmp/orig.so $lib
