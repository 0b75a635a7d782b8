# round-2 v7 verification at HEAD: default (c4) and c2 bench lines first, then smoke and the GPU suite
timeout 900 python bench.py > gpurun_out/z_c4_bench.json 2> gpurun_out/z_c4_bench.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/z_c2_bench.json 2> /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/z_pytest_gpu.txt 2>&1
