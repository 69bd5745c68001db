timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c2.json')); print(d['value'], d['roofline']['avg_kernel_ms'], d['roofline']['frac'])"
FRAMES=512 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sobel_tma -s 1 -c 1 -o gpurun_out/r02_sobel_tma_h2 python tools/sobel_sweep.py > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log
