# HEAD verification on the B200: GPU tests, smoke, default (c4) bench line, c2 line
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/v5_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v5_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/v5_c4.json 2> gpurun_out/v5_c4.err
timeout 300 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/v5_c2.json 2> gpurun_out/v5_c2.err
