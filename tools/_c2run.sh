timeout 900 python -m pytest tests/test_gpu_resident_widths.py tests/test_gpu_helmholtz.py tests/test_gpu_fuzz.py tests/test_gpu_large.py tests/test_gpu_loop_modes.py -q -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed" | head -20
timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 > gpurun_out/r02_bench_c1.json 2>gpurun_out/r02_bench_c1.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c1.json')); print(d['value']/1e9, d['ms_per_step'], d['roofline']['avg_kernel_ms'], d['e2e']['value']/1e9)"
