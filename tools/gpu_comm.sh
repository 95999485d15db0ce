set -x
timeout 300 python -m pytest tests/test_gpu_comm_report.py -x -q 2>&1 | tail -3
timeout 1500 python -m paper_2512_20017_b200.comm_report --config c4 --gpus 2 4 8 --out gpurun_out/comm_c4.json > gpurun_out/comm_c4.log 2>&1; tail -5 gpurun_out/comm_c4.log
timeout 2400 python -m paper_2512_20017_b200.comm_report --config c5 --gpus 8 --out gpurun_out/comm_c5.json > gpurun_out/comm_c5.log 2>&1; tail -5 gpurun_out/comm_c5.log
