python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu_r2a.txt 2>&1
python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_r2a.json 2> gpurun_out/bench_c2_r2a.err
