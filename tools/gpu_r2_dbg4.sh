# the lagging-rank test against a build without the exit wait (shipped in the checked slot)
OSP_LIB_VARIANT=checked timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "lagging" 2>&1 | grep -E "AssertionError: |passed|failed" | head -5
