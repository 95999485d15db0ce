# bench C2 under several nvcc -D flag sets: FLAGS="A|B|C" (| separated), default build last
IFS='|' read -ra SETS <<< "${FLAGS}"
for F in "${SETS[@]}" ""; do
  BS_NVCC_EXTRA="$F" python -m paper_2512_20017_b200.build -f > /dev/null 2>&1
  timeout 300 python bench.py --config ${CFG:-c2} --no-cpu-baseline --steps 20 > gpurun_out/sweep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep.json')); print('[$F]', d['value'], {k:v['ms'] for k,v in d['stages'].items()})"
done
