# round-2 v4 measurement set at HEAD: GPU suite, smoke, bench lines c1-c5, c4/c2 launch lists, c4 tensor pipe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/x_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/x_c4_bench.json 2> gpurun_out/x_c4_bench.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/x_c2_bench.json 2> /dev/null
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/x_c5_bench.json 2> /dev/null
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --graph > gpurun_out/x_c1_bench.json 2> /dev/null
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --metamer 100 > gpurun_out/x_c3_bench.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/x_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/x_c2_launches.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_joint --csv --log-file gpurun_out/x_c4_tensor.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/x_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.txt 2>&1
