timeout 900 python -m pytest tests/test_gpu_densify_multirank.py -x -q 2>&1 | tail -15
