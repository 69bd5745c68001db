timeout 900 python -m pytest tests/test_gpu_reduce_fold.py tests/test_gpu_jit.py tests/test_gpu_partition_sets.py -q -p no:cacheprovider 2>&1 | grep -E "^E  |passed|failed|FAILED" | head -30
