python tools/_dbg_prefetch.py
timeout 900 python -m pytest tests/test_gpu_resident_widths.py tests/test_gpu_prefetch.py -q -p no:cacheprovider 2>&1 | tail -8
