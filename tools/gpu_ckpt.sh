timeout 900 python -m pytest tests/test_gpu_densify.py tests/test_gpu_fused_adam.py -x -q 2>&1 | tail -5
