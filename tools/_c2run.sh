timeout 900 python -m pytest tests/test_gpu_stream_farm.py tests/test_streams.py tests/test_gpu_apps.py -q -p no:cacheprovider 2>&1 | tail -2
