timeout 900 python -m pytest tests/test_gpu_stream_farm.py tests/test_gpu_apps.py tests/test_gpu_split_restore.py tests/test_streams.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 > gpurun_out/r02_bench_c2.json 2>gpurun_out/r02_bench_c2.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c2.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['passes_frames_per_s'])"; tail -2 gpurun_out/r02_bench_c2.err
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > gpurun_out/r02_bench_c5.json 2>gpurun_out/r02_bench_c5.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c5.json')); print(d['value'], d['e2e']['value'], d['e2e']['passes_frames_per_s'])"; tail -2 gpurun_out/r02_bench_c5.err
