timeout 600 python -m pytest tests/test_gpu_sobel_tma.py tests/test_gpu_large.py -k "sobel" tests/test_gpu_apps.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in 0 1 5 6; do SK_TMA_CFG=$c python tools/sobel_sweep.py; done
