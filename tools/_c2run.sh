SK_HELM_TMA=2 timeout 900 python -m pytest tests/test_gpu_helmholtz.py tests/test_gpu_production.py tests/test_gpu_fuzz.py tests/test_gpu_resident_widths.py -q -x -p no:cacheprovider 2>&1 | tail -3
SK_HELM_TMA=1 python tools/prof_helmholtz.py --n 23170 --dtype f64 --solves 2 | tail -1
python tools/prof_helmholtz.py --n 23170 --dtype f64 --solves 2 | tail -1
