timeout 900 python -m pytest tests/test_gpu_split_restore.py tests/test_gpu_stream_farm.py tests/test_gpu_apps.py tests/test_native_abi.py -q -x -p no:cacheprovider 2>&1 | tail -25
