for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "oversubscribed_ragged and 2-4-1.0" 2>&1 | grep -E "Error|assert|passed|failed|rank" | head -20; done
