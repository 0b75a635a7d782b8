python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/hw_tests.txt
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hw.json
timeout 300 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/dram_all.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dram_all.log 2>&1
